"""Domain decomposition host logic ("next").

North_star runs one GPU with no sharding, so this module is the host half of
the multi-GPU step only: the SFC split of the cells, the rank-boundary face
lists both sides derive identically, the skeleton rule widened by rank
boundaries, and the per-step exchange plumbing (face traces to each
neighbour rank, dt as a global MIN) over `torch.distributed`.

Reference anchors:
  * `decomp.rank_of(key)` / `decomp.nranks` / `decomp.version` as consumed by
    `mesh.py:537-567` (secondary_order) and `mesh.py:599-610`;
  * `classify_cell(mesh, node, decomp)` `mesh.py:585-596` -- a cell that
    touches a rank boundary is skeleton;
  * `boundary_face_order(mesh, decomp, rank_pair)` `mesh.py:613-628` -- the
    shared faces of a rank pair, the same list from either rank, ConfigError
    on an unknown pair;
  * SPEC.md:425-508 (rank-sim): `decompose(mesh, R)` splits the SFC order
    into R contiguous segments whose cell counts differ by at most one,
    ConfigError for R outside [1, ncells].

B200 design choice: the reference sends one message per face (SPEC.md
rank-sim "deliberately per-face"); over NVLink a message costs launch
latency, not bandwidth, so `exchange_traces` sends ONE contiguous buffer per
neighbour rank per step, laid out in boundary_face_order, so the receiver's
rows line up with its own boundary-face list without an index map.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import ConfigError
from .mesh import AdaptiveMesh, CartesianMesh


def _morton3_key(idx, depth):
    """Morton order over the 3-ary index space (SPEC.md rank-sim design
    decisions): the level-l digit of every axis, coarsest level first."""
    return tuple(tuple((i // 3 ** (depth - l)) % 3 for i in idx) for l in range(1, depth + 1))


def _depth(N):
    """Tree depth of an N-per-axis uniform mesh (N = 3^depth for the reference's meshes)."""
    depth = 1
    while 3 ** depth < N:
        depth += 1
    return depth


def sfc_order(mesh):
    """Cell indices of `mesh` in space-filling-curve order."""
    if isinstance(mesh, AdaptiveMesh):
        return np.arange(mesh.ncells, dtype=np.int64)   # cells are stored in SFC order
    if isinstance(mesh, CartesianMesh):
        depth = _depth(mesh.N)
        keys = [_morton3_key(tuple(int(v) for v in row), depth) for row in mesh.index]
        return np.array(sorted(range(mesh.ncells), key=keys.__getitem__), dtype=np.int64)
    raise ConfigError(f"unsupported mesh type {type(mesh).__name__}")


def interior_faces(mesh):
    """(F, 2) int64 owner cells (lo, hi) of every leaf face between two
    distinct real cells, in the mesh's canonical face order, plus each face's
    sort key (axis, level, position) -- the reference FaceRecord.key,
    `mesh.py:92-94`.  Domain-boundary faces are excluded; a hanging child
    face lists its coarse owner on the virtual side."""
    if isinstance(mesh, AdaptiveMesh):
        keep = (mesh.face_kind != 2).all(axis=1) & (mesh.face_cell[:, 0] != mesh.face_cell[:, 1])
        keys = [(k[1], k[2], k[3]) for k, ok in zip(mesh._leaf_keys, keep) if ok]
        return mesh.face_cell[keep].astype(np.int64), keys
    if isinstance(mesh, CartesianMesh):
        # FaceRecord.key of the reference uniform mesh: (axis, level, index of
        # the upper cell), which wraps to 0 along the axis on a periodic face
        depth = _depth(mesh.N)
        out, keys = [], []
        for a in range(mesh.dim):
            hi = mesh.nbr[:, 2 * a + 1].astype(np.int64)
            lo = np.arange(mesh.ncells, dtype=np.int64)
            ok = (hi >= 0) & (hi != lo)
            out.append(np.stack([lo[ok], hi[ok]], axis=1))
            keys.extend((a, depth, tuple(int(v) for v in mesh.index[c])) for c in hi[ok])
        return np.concatenate(out, axis=0), keys
    raise ConfigError(f"unsupported mesh type {type(mesh).__name__}")


@dataclass
class DomainDecomposition:
    """Cell -> rank map from contiguous cuts of the SFC order."""
    nranks: int
    cell_rank: np.ndarray          # (ncells,) int32
    version: int = 0

    def rank_of(self, cell):
        return int(self.cell_rank[cell])

    def cells_of(self, rank):
        return np.nonzero(self.cell_rank == rank)[0].astype(np.int32)


def decompose(mesh, nranks: int) -> DomainDecomposition:
    """SPEC.md rank-sim `decompose`: R contiguous SFC segments, sizes differ by <= 1
    (the first ncells % R segments hold one extra cell)."""
    n = mesh.ncells
    if not (1 <= nranks <= n):
        raise ConfigError(f"rank count {nranks} outside [1, {n}]")
    order = sfc_order(mesh)
    base, extra = divmod(n, nranks)
    sizes = np.full(nranks, base, dtype=np.int64)
    sizes[:extra] += 1
    seg = np.repeat(np.arange(nranks, dtype=np.int32), sizes)
    cell_rank = np.empty(n, dtype=np.int32)
    cell_rank[order] = seg
    return DomainDecomposition(nranks, cell_rank, version=getattr(mesh, "version", 0))


def boundary_face_order(mesh, decomp: DomainDecomposition, rank_pair):
    """Indices into `interior_faces(mesh)` of the faces shared by the two
    ranks, identical from either rank, in the reference's secondary-sweep
    order (`mesh.py:552-564`, `mesh.py:613-628`): a face is emitted after the
    later of its two owners in SFC order, ties broken by face key."""
    r1, r2 = rank_pair
    if not (0 <= r1 < decomp.nranks and 0 <= r2 < decomp.nranks):
        raise ConfigError(f"unknown rank pair {rank_pair}")
    if r1 == r2:
        return np.zeros(0, dtype=np.int64)
    faces, keys = interior_faces(mesh)
    ra, rb = decomp.cell_rank[faces[:, 0]], decomp.cell_rank[faces[:, 1]]
    sel = np.nonzero(((ra == r1) & (rb == r2)) | ((ra == r2) & (rb == r1)))[0]
    pos = np.empty(mesh.ncells, dtype=np.int64)
    pos[sfc_order(mesh)] = np.arange(mesh.ncells)
    later = np.maximum(pos[faces[:, 0]], pos[faces[:, 1]])
    return np.array(sorted(sel.tolist(), key=lambda f: (int(later[f]), keys[f])), dtype=np.int64)


def skeleton_mask(mesh, decomp: DomainDecomposition | None):
    """`classify_cell` with a decomposition (`mesh.py:585-596`): skeleton iff
    one of the cell's sides is a parent face (the coarse side of a
    resolution transition) or a face below it joins cells on two ranks.
    (Config 5's schedule rule, `AdaptiveMesh.skeleton_mask`, also marks the
    fine side and the synthetic cut.)"""
    if isinstance(mesh, AdaptiveMesh):
        mask = (mesh.side_face >= mesh.nleaf).any(axis=1)
    else:
        mask = np.zeros(mesh.ncells, dtype=bool)
    if decomp is not None:
        faces, _ = interior_faces(mesh)
        cross = decomp.cell_rank[faces[:, 0]] != decomp.cell_rank[faces[:, 1]]
        mask[faces[cross].ravel()] = True
    return mask


@dataclass
class ExchangePlan:
    """Per-rank view: for each neighbour rank, the shared faces (indices into
    interior_faces) and, per face, this rank's local owner cell and the
    side (0 = lo, 1 = hi) that cell occupies.

    Hanging faces (AdaptiveMesh): the payload of a face is always the local
    owner's whole side trace (`local_fs`); when the local owner is the coarse
    cell of a chain, the RECEIVER evaluates it at the leaf face's points with
    the face's interpolation path (`vpath` / `vdepth`, coarsest level first,
    the same path the device face kernel applies), exactly as it would for a
    local coarse neighbour -- the reference sends the projection from the
    local adjacent cell, which for the coarse owner is that
    trace."""
    rank: int
    peers: list
    faces: dict          # peer -> (k,) int64 face indices in boundary_face_order
    local_cell: dict     # peer -> (k,) int64 cell owned by `rank`
    local_side: dict     # peer -> (k,) int8
    local_fs: dict       # peer -> (k,) int8: the local cell's side slot 2*axis + s of the face
    vpath: dict = field(default_factory=dict)    # peer -> (k, MAX_CHAIN, 2) int8 (AdaptiveMesh)
    vdepth: dict = field(default_factory=dict)   # peer -> (k,) int8: 0 = no virtual side
    device_index: dict = field(default_factory=dict)   # (peer, device) -> (cell int32, fs int8) on the device


def exchange_plan(mesh, decomp: DomainDecomposition, rank: int) -> ExchangePlan:
    faces, keys = interior_faces(mesh)
    axis = np.array([k[0] for k in keys], dtype=np.int64)
    peers, fmap, cmap, smap, fsmap = [], {}, {}, {}, {}
    for q in range(decomp.nranks):
        if q == rank:
            continue
        f = boundary_face_order(mesh, decomp, (rank, q))
        if f.size == 0:
            continue
        lo_mine = decomp.cell_rank[faces[f, 0]] == rank
        peers.append(q)
        fmap[q] = f
        cmap[q] = np.where(lo_mine, faces[f, 0], faces[f, 1])
        smap[q] = np.where(lo_mine, 0, 1).astype(np.int8)
        # the lo owner sees the face on its upper side (s = 1), the hi owner on its lower side
        fsmap[q] = (2 * axis[f] + np.where(lo_mine, 1, 0)).astype(np.int8)
    plan = ExchangePlan(rank, peers, fmap, cmap, smap, fsmap)
    if isinstance(mesh, AdaptiveMesh):
        leaf = np.nonzero((mesh.face_kind != 2).all(axis=1) & (mesh.face_cell[:, 0] != mesh.face_cell[:, 1]))[0]
        for q in peers:
            li = leaf[fmap[q]]
            plan.vpath[q] = mesh.face_vpath[li].copy()
            plan.vdepth[q] = np.where((mesh.face_kind[li] == 1).any(axis=1), mesh.face_vdepth[li], 0).astype(np.int8)
    return plan


def pack_boundary_traces(plan: ExchangePlan, peer: int, trace_q, trace_f):
    """Send buffer (k, 2, m*n^(d-1)) for `peer` gathered on the device by
    `edg_pack_face_traces` from the STP traces (C, 2d, m, n^(d-1))."""
    import torch
    from . import _lib
    from .kernels import _stream
    for t, nm in ((trace_q, "trace_q"), (trace_f, "trace_f")):
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
            raise ConfigError(f"{nm} must be a contiguous float64 CUDA tensor")
    if trace_q.shape != trace_f.shape or trace_q.device != trace_f.device or trace_q.dim() < 3:
        raise ConfigError("trace_q and trace_f must have the same (C, 2d, m, ...) shape on one device")
    if peer not in plan.local_cell:
        raise ConfigError(f"rank {peer} is not a neighbour of rank {plan.rank}")
    C_, nsides = trace_q.shape[0], trace_q.shape[1]
    row_len = trace_q[0, 0].numel()
    dev = trace_q.device
    key = (peer, str(dev))
    if key not in plan.device_index:     # uploaded once per plan, not per step
        plan.device_index[key] = (torch.from_numpy(plan.local_cell[peer].astype(np.int32)).to(dev),
                                  torch.from_numpy(plan.local_fs[peer]).to(dev))
    cell, side = plan.device_index[key]
    out = torch.empty((cell.numel(), 2, row_len), dtype=torch.float64, device=dev)
    _lib.check(_lib.load().edg_pack_face_traces(nsides, row_len, cell.numel(), _lib.ptr(cell), _lib.ptr(side),
                                                _lib.ptr(trace_q), _lib.ptr(trace_f), _lib.ptr(out),
                                                _stream()), "pack face traces")
    return out


def unpack_boundary_traces(recv, slots, ghost):
    """Scatter received rows (k, 2, L) into ghost[slots] (G, 2, L) on the device
    (`slots`: host ints, or a resident int32 device tensor)."""
    import torch
    from . import _lib
    from .kernels import _stream
    for t, nm in ((recv, "recv"), (ghost, "ghost")):
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
            raise ConfigError(f"{nm} must be a contiguous float64 CUDA tensor")
    if recv.dim() != 3 or ghost.dim() != 3 or recv.shape[1] != 2 or ghost.shape[1] != 2 or \
            recv.shape[2] != ghost.shape[2] or recv.device != ghost.device:
        raise ConfigError(f"recv {tuple(recv.shape)} / ghost {tuple(ghost.shape)}: expected (k, 2, L) / (G, 2, L)")
    if isinstance(slots, torch.Tensor):
        slot = slots.to(device=ghost.device, dtype=torch.int32).contiguous()
    else:
        slot = torch.as_tensor(np.asarray(slots, dtype=np.int32)).to(ghost.device)
    if slot.numel() != recv.shape[0]:
        raise ConfigError(f"{slot.numel()} slots for {recv.shape[0]} received rows")
    if slot.numel() and (int(slot.min()) < 0 or int(slot.max()) >= ghost.shape[0]):
        raise ConfigError(f"ghost slot outside [0, {ghost.shape[0]})")
    _lib.check(_lib.load().edg_unpack_face_traces(recv.shape[-1], recv.shape[0], _lib.ptr(slot), _lib.ptr(recv),
                                                  _lib.ptr(ghost), _stream()), "unpack face traces")
    return ghost


def exchange_traces(dist, plan: ExchangePlan, send: dict):
    """Send `send[peer]` (rows in the peer's boundary_face_order) to every
    peer and return {peer: received rows}.  One message per neighbour per
    step; tensors may live on the GPU (NCCL) or the CPU (gloo)."""
    import torch
    reqs, recv = [], {}
    for q in plan.peers:
        buf = send[q]
        if buf.shape[0] != plan.faces[q].shape[0]:
            raise ConfigError(f"payload for rank {q} has {buf.shape[0]} rows, expected {plan.faces[q].shape[0]}")
        recv[q] = torch.empty_like(buf)
    for q in plan.peers:
        # lower rank sends first so the pairwise order never deadlocks on blocking backends
        if plan.rank < q:
            reqs.append(dist.isend(send[q].contiguous(), q))
            reqs.append(dist.irecv(recv[q], q))
        else:
            reqs.append(dist.irecv(recv[q], q))
            reqs.append(dist.isend(send[q].contiguous(), q))
    for r in reqs:
        r.wait()
    return recv


def global_dt(dist, local_candidate, cfl=1.0):
    """Admissible dt of the whole domain (kernels.py:267-281 over all ranks):
    all-reduce MIN of each rank's raw candidate min_c h_c / ((2p+1) lambda_c)
    -- None or +inf for a rank without a positive wave speed -- THEN the cfl
    factor, so the result is bitwise the single-domain one and a quiet rank
    cannot poison it.  Raises EnclaveDgError only when no rank has a
    candidate.  The reduction tensor lives on the backend's device (CUDA for
    NCCL).  The device path of the sharded step all-reduces the 256 dt slots
    instead (sharded.ShardedDGSolver)."""
    import torch
    from .errors import EnclaveDgError
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu")
    if isinstance(local_candidate, torch.Tensor):
        t = local_candidate.detach().to(device=dev, dtype=torch.float64).reshape(1).clone()
    else:
        v = float("inf") if local_candidate is None else float(local_candidate)
        t = torch.tensor([v], dtype=torch.float64, device=dev)
    t = torch.where(torch.isnan(t) | (t <= 0), torch.full_like(t, float("inf")), t)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    best = float(t.item())
    if best == float("inf"):
        raise EnclaveDgError("no positive wave speed anywhere; cannot pick a time step")
    return float(cfl) * best
