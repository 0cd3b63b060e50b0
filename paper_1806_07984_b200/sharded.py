"""Sharded ADER-DG step: one rank's share of a decomposed uniform mesh
(SPEC.md:425-508 rank-sim).

Per rank and step (the paper's MPI+X scheme on the device):

    main:  all-reduce MIN of the dt candidate slots over the ranks -> dt
    high:  predictor of the skeleton cells (cells with a face on another rank)
           -> pack their boundary face traces (one buffer per neighbour rank,
           rows in boundary_face_order) -> exchange -> unpack into ghost rows
    low:   predictor of the enclave cells (overlaps the exchange)
    main:  fused Riemann + corrector over the local cells, reading a remote
           neighbour's trace from its ghost row (+ next dt candidates)

Every face on a rank boundary is solved redundantly by both owners from the
same two traces with the same operation order, so the two outcomes are
bitwise equal ("redundant-solve agreement"), and the whole
decomposed run is bitwise the single-domain run ("rank-count
transparency"; tests/test_gpu_sharded.py).  Only the time-integrated face
trace `trace_q` crosses ranks (the reference's "Q*_h projection",
SPEC.md:455): the owner's `trace_f` is never needed by the other side.

The dt candidates are exchanged as their 256 device slots (positive doubles
ordered by their bits; the empty slot is INT64_MAX), so one int64 MIN
all-reduce yields exactly the single-domain minimum, and a rank without any
positive wave speed cannot poison it (the reference raises only when the
whole domain has none, kernels.py:279-280).

Communication goes through a `comm` object: `TorchComm` (torch.distributed:
NCCL on device buffers, gloo through host staging) or `LoopbackComm`
(ranks emulated one after another in one process, the SPEC's "interleaved"
rank mode).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .basis import get_basis
from .decomposition import DomainDecomposition, exchange_plan, interior_faces
from .errors import ConfigError
from .kernels import _check_supported, _stream, _torch
from .mesh import CartesianMesh
from .pde import PdeDescriptor
from .solver import _Base


@dataclass
class ShardLayout:
    """Host-side index maps of one rank (numpy only).

    local:     (L,) global ids of the owned cells (ascending)
    ghost:     (G,) global ids of the remote face neighbours (ascending)
    nbr:       (L, 2d) int32 neighbour of each local cell side in the local
               numbering [local | ghost], -1 = outflow boundary
    skeleton / enclave: local indices of the cells with / without a remote neighbour
    peers:     neighbour ranks
    send_rows: {peer: (k,) int64 row = local_cell * 2d + side slot}, rows in
               boundary_face_order of the pair (what this rank sends)
    recv_rows: {peer: (k,) int64 row = (L + ghost_pos) * 2d + side slot of the
               remote cell}, same order (where the received rows go)
    """
    rank: int
    nranks: int
    local: np.ndarray
    ghost: np.ndarray
    nbr: np.ndarray
    skeleton: np.ndarray
    enclave: np.ndarray
    peers: list
    send_rows: dict
    recv_rows: dict


def shard_layout(mesh: CartesianMesh, decomp: DomainDecomposition, rank: int) -> ShardLayout:
    if not isinstance(mesh, CartesianMesh):
        raise ConfigError("the sharded step supports Cartesian meshes")
    if not 0 <= rank < decomp.nranks:
        raise ConfigError(f"rank {rank} outside [0, {decomp.nranks})")
    d2 = 2 * mesh.dim
    local = decomp.cells_of(rank).astype(np.int64)
    L = local.size
    gnbr = mesh.nbr[local].astype(np.int64)                       # (L, 2d) global
    remote = (gnbr >= 0) & (decomp.cell_rank[np.maximum(gnbr, 0)] != rank)
    ghost = np.unique(gnbr[remote])
    g2l = np.full(mesh.ncells, -1, dtype=np.int64)
    g2l[local] = np.arange(L)
    g2l[ghost] = L + np.arange(ghost.size)
    nbr = np.where(gnbr >= 0, g2l[np.maximum(gnbr, 0)], -1).astype(np.int32)
    skel = remote.any(axis=1)
    plan = exchange_plan(mesh, decomp, rank)
    faces, _ = interior_faces(mesh)
    send_rows, recv_rows = {}, {}
    for q in plan.peers:
        f = plan.faces[q]
        mine = plan.local_cell[q].astype(np.int64)
        other = np.where(faces[f, 0] == mine, faces[f, 1], faces[f, 0])
        fs = plan.local_fs[q].astype(np.int64)
        send_rows[q] = g2l[mine] * d2 + fs
        recv_rows[q] = g2l[other] * d2 + (fs ^ 1)                 # the remote cell sees the face on the other side
    return ShardLayout(rank, decomp.nranks, local, ghost, nbr, np.nonzero(skel)[0].astype(np.int32),
                       np.nonzero(~skel)[0].astype(np.int32), list(plan.peers), send_rows, recv_rows)


# ------------------------------------------------------------------ comms --

class TorchComm:
    """torch.distributed transport: device buffers on NCCL, host staging on gloo."""

    def __init__(self, dist):
        self.dist = dist
        self.staged = dist.get_backend() != "nccl"

    def allreduce_min_(self, t):
        if self.staged:
            h = t.cpu()
            self.dist.all_reduce(h, op=self.dist.ReduceOp.MIN)
            t.copy_(h)
        else:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN)

    def exchange(self, rank, send: dict, recv: dict):
        """send[peer] -> peer, recv[peer] <- peer; lower rank posts its send first."""
        import torch
        dist = self.dist
        bufs = {q: (send[q].cpu() if self.staged else send[q]) for q in send}
        rbufs = {q: (torch.empty(recv[q].shape, dtype=recv[q].dtype) if self.staged else recv[q]) for q in recv}
        reqs = []
        for q in sorted(send):
            if rank < q:
                reqs += [dist.isend(bufs[q], q), dist.irecv(rbufs[q], q)]
            else:
                reqs += [dist.irecv(rbufs[q], q), dist.isend(bufs[q], q)]
        for r in reqs:
            r.wait()
        if self.staged:
            for q in recv:
                recv[q].copy_(rbufs[q])


class LoopbackComm:
    """In-process rank emulation: `ShardedDGSolver.emulate_step` drives the
    ranks phase by phase and moves the buffers directly."""


# ----------------------------------------------------------------- solver --

class ShardedDGSolver(_Base):
    """One rank of a decomposed uniform-mesh ADER-DG run (see module doc)."""

    def __init__(self, pde: PdeDescriptor, order: int, mesh: CartesianMesh, cfl: float,
                 decomp: DomainDecomposition, rank: int, comm=None, tol: float = 1e-10, max_iter=None,
                 check_finite: bool = True, max_steps: int = 4096, two_streams: bool = True):
        torch = self.torch = _torch()
        self.lib = _lib.load()
        _check_supported(pde, order)
        if mesh.dim != pde.dim:
            raise ConfigError("mesh and pde dimension differ")
        self.pde, self.order, self.mesh, self.cfl = pde, order, mesh, float(cfl)
        self.tol, self.max_iter = float(tol), 0 if max_iter is None else int(max_iter)
        self.check_finite = check_finite
        self.decomp, self.rank, self.comm = decomp, rank, comm
        self.basis = get_basis(order)
        self.table = self.basis.device_table()
        self.native = pde.native()
        self.layout = lay = shard_layout(mesh, decomp, rank)
        d, m, n = pde.dim, pde.m, self.basis.n
        L, G = lay.local.size, lay.ghost.size
        self.ncells, self.nghost = L, G
        f64 = dict(dtype=torch.float64, device="cuda")
        i32 = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).cuda()  # noqa: E731
        i64 = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.int64)).cuda()  # noqa: E731
        self.Q = torch.zeros((L, m) + (n,) * d, **f64)
        self.Qn = torch.zeros_like(self.Q)
        self.q_end = torch.zeros_like(self.Q)
        self.trace_q = torch.zeros((L + G, 2 * d, m) + (n,) * (d - 1), **f64)   # local rows, then ghost rows
        self.trace_f = torch.zeros((L, 2 * d, m) + (n,) * (d - 1), **f64)
        self.row_len = m * n ** (d - 1)
        self.iterations = torch.zeros(L, dtype=torch.int32, device="cuda")
        self.converged = torch.zeros(L, dtype=torch.uint8, device="cuda")
        self.iter_total = torch.zeros(1, dtype=torch.int64, device="cuda")
        self._common_alloc(max_steps)
        self.edges = torch.tensor([mesh.h] * d, **f64)
        self.hmin = torch.tensor([mesh.h], **f64)
        self.nbr = i32(lay.nbr)
        self.skel, self.encl = i32(lay.skeleton), i32(lay.enclave)
        self.send_rows = {q: i64(r) for q, r in lay.send_rows.items()}
        self.recv_rows = {q: i64(r) for q, r in lay.recv_rows.items()}
        self.send = {q: torch.empty((r.size, self.row_len), **f64) for q, r in lay.send_rows.items()}
        self.recv = {q: torch.empty((r.size, self.row_len), **f64) for q, r in lay.recv_rows.items()}
        self.two_streams = two_streams
        if two_streams:
            lo, hi = C.c_int32(), C.c_int32()
            _lib.check(self.lib.edg_stream_priority_range(C.byref(lo), C.byref(hi)), "priority range")
            self.s_hi = torch.cuda.Stream(priority=hi.value)
            self.s_lo = torch.cuda.Stream(priority=lo.value)

    # ------------------------------------------------------------- state --
    def set_state(self, Q_global):
        """Take this rank's cells out of a global (C, m, n^d) state."""
        torch = self.torch
        src = Q_global if isinstance(Q_global, torch.Tensor) else torch.from_numpy(
            np.ascontiguousarray(Q_global, dtype=np.float64))
        idx = torch.from_numpy(self.layout.local)
        self.Q.copy_(src.reshape((-1,) + tuple(self.Q.shape[1:]))[idx.to(src.device)], non_blocking=True)
        self.steps_done = 0
        self.status.zero_()
        _lib.check(self.lib.edg_dt_slots_reset(_lib.ptr(self.slots), _stream()), "dt reset")
        _lib.check(self.lib.edg_cell_speed_reduce(C.byref(self.native), self.order, self.ncells,
                                                  self.basis.n ** self.pde.dim, _lib.ptr(self.Q), _lib.ptr(self.hmin),
                                                  0, _lib.ptr(self.slots), _stream()), "admissible_dt")

    def state(self):
        return self.Q

    # ------------------------------------------------------------ phases --
    def _stp(self, cells, background=False):
        if cells.numel() == 0:
            return
        fn = self.lib.edg_stp_picard_background if background else self.lib.edg_stp_picard
        _lib.check(fn(C.byref(self.native), self.order, _lib.ptr(self.table), _lib.ptr(self.Q),
                                           _lib.ptr(cells), int(cells.numel()), _lib.ptr(self.edges), 0,
                                           _lib.ptr(self.dt), self.tol, self.max_iter, _lib.ptr(self.q_end), None,
                                           _lib.ptr(self.trace_q), _lib.ptr(self.trace_f),
                                           _lib.ptr(self.iterations), _lib.ptr(self.converged),
                                           _lib.ptr(self.iter_total), _stream()), "stp_picard")

    def _pack(self):
        rows = self.trace_q.view(-1, self.row_len)
        for q, idx in self.send_rows.items():
            _lib.check(self.lib.edg_gather_rows(self.row_len, int(idx.numel()), _lib.ptr(idx), _lib.ptr(rows),
                                                _lib.ptr(self.send[q]), _stream()), "pack")

    def _unpack(self):
        rows = self.trace_q.view(-1, self.row_len)
        for q, idx in self.recv_rows.items():
            _lib.check(self.lib.edg_scatter_rows(self.row_len, int(idx.numel()), _lib.ptr(idx), _lib.ptr(self.recv[q]),
                                                 _lib.ptr(rows), _stream()), "unpack")

    def _correct(self):
        _lib.check(self.lib.edg_corrector(C.byref(self.native), self.order, _lib.ptr(self.table), self.ncells,
                                          _lib.ptr(self.q_end), _lib.ptr(self.trace_q), _lib.ptr(self.trace_f),
                                          _lib.ptr(self.nbr), None, None, _lib.ptr(self.edges), 0,
                                          _lib.ptr(self.Qn), _lib.ptr(self.slots), _lib.ptr(self.hmin),
                                          _lib.ptr(self.status), _stream()), "corrector")
        self.Q, self.Qn = self.Qn, self.Q

    def predict(self):
        """dt from the (already globally reduced) slots, predictors, pack (one stream)."""
        self._finalize_dt()
        self._stp(self.skel)
        self._pack()
        self._stp(self.encl)

    def finish(self):
        """Unpack the received traces and correct (one stream)."""
        self._unpack()
        self._correct()
        self.steps_done += 1

    # -------------------------------------------------------------- step --
    def step(self):
        """One step with a torch.distributed transport (`comm` = TorchComm)."""
        torch = self.torch
        if not isinstance(self.comm, TorchComm):
            raise ConfigError("step() needs a TorchComm; emulated ranks go through emulate_step")
        self.comm.allreduce_min_(self.slots)
        self._finalize_dt()
        if not self.two_streams:
            self._stp(self.skel)
            self._pack()
            self.comm.exchange(self.rank, self.send, self.recv)
            self._stp(self.encl)
            self.finish()
            return
        main = torch.cuda.current_stream()
        self.s_hi.wait_stream(main)
        self.s_lo.wait_stream(main)
        with torch.cuda.stream(self.s_hi):
            self._stp(self.skel)
            self._pack()
            self.comm.exchange(self.rank, self.send, self.recv)
            self._unpack()
        with torch.cuda.stream(self.s_lo):
            self._stp(self.encl, background=True)
        main.wait_stream(self.s_hi)
        main.wait_stream(self.s_lo)
        self._correct()
        self.steps_done += 1

    @staticmethod
    def emulate_step(ranks):
        """One step of all ranks in one process (SPEC.md:500 interleaved mode):
        dt slots combined by MIN, each rank predicts and packs, the buffers
        move rank to rank, each rank unpacks and corrects."""
        torch = _torch()
        lo = torch.stack([r.slots for r in ranks]).min(dim=0).values
        for r in ranks:
            r.slots.copy_(lo)
        for r in ranks:
            r.predict()
        for r in ranks:
            for q in r.layout.peers:
                r.recv[q].copy_(ranks[q].send[r.rank])
        for r in ranks:
            r.finish()

    def gather_into(self, Q_global):
        """Write this rank's cells into a global (C, m, n^d) device tensor."""
        torch = self.torch
        Q_global[torch.from_numpy(self.layout.local).to(Q_global.device)] = self.Q
        return Q_global
