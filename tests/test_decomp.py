"""Row f3 host logic: SFC decomposition, rank-boundary face order, skeleton
rule with ranks (pinned to the reference mesh through tests/golden/decomp.json,
made by tests/golden/make_golden_decomp.py), and the per-neighbour trace
exchange + dt all-reduce over gloo with world size 2."""
import json
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1806_07984_b200.decomposition import (boundary_face_order, decompose, exchange_plan, interior_faces,
                                                 skeleton_mask)
from paper_1806_07984_b200.errors import ConfigError
from paper_1806_07984_b200.mesh import AdaptiveMesh, CartesianMesh

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "decomp.json")))


def _key(k):
    return tuple(tuple(x) if isinstance(x, list) else x for x in k)


@pytest.mark.parametrize("name,N", [("uniform3", 3), ("uniform9", 9)])
def test_cartesian_against_reference_mesh(name, N):
    """A periodic CartesianMesh decomposes like the reference's uniform mesh:
    same partition, same boundary faces in the same order (face keys
    (axis, level, upper cell index) with the periodic wrap), same skeleton."""
    G = GOLDEN[name]
    mesh = CartesianMesh(N, 2, True)
    level = G["cells"][0][0]
    key_of = {(level, tuple(int(v) for v in mesh.index[c])): c for c in range(mesh.ncells)}
    faces, fkeys = interior_faces(mesh)
    for case in G["cases"]:
        R = case["R"]
        dec = decompose(mesh, R)
        for pair, want in case["pairs"].items():
            r1, r2 = map(int, pair.split(","))
            got = boundary_face_order(mesh, dec, (r1, r2))
            assert list(got) == list(boundary_face_order(mesh, dec, (r2, r1)))
            got_t = [(faces[f, 0], faces[f, 1], fkeys[f]) for f in got]
            want_t = [(key_of[_key(lo)], key_of[_key(hi)], _key(fk)) for lo, hi, fk in want]
            assert got_t == want_t, (R, pair)
        skel = set(np.nonzero(skeleton_mask(mesh, dec))[0].tolist())
        assert skel == {key_of[_key(c)] for c in case["skeleton"]}


@pytest.mark.parametrize("name", ["uniform3", "uniform9", "refined"])
def test_against_reference_mesh(name):
    G = GOLDEN[name]
    cells = [_key(c) for c in G["cells"]]
    mesh = AdaptiveMesh(cells, 2, True)
    assert mesh.cells == cells                      # same SFC order as the reference
    faces, fkeys = interior_faces(mesh)
    for case in G["cases"]:
        R = case["R"]
        dec = decompose(mesh, R)
        sizes = np.bincount(dec.cell_rank, minlength=R)
        assert sizes.max() - sizes.min() <= 1
        for pair, want in case["pairs"].items():
            r1, r2 = map(int, pair.split(","))
            got = boundary_face_order(mesh, dec, (r1, r2))
            assert list(got) == list(boundary_face_order(mesh, dec, (r2, r1)))
            got_t = [(cells[faces[f, 0]], cells[faces[f, 1]], fkeys[f]) for f in got]
            want_t = [(_key(lo), _key(hi), _key(fk)) for lo, hi, fk in want]
            assert got_t == want_t
        skel = {cells[i] for i in np.nonzero(skeleton_mask(mesh, dec))[0]}
        assert skel == {_key(c) for c in case["skeleton"]}


def test_decompose_examples():
    m81 = CartesianMesh(9, 2, True)
    d1 = decompose(m81, 1)
    assert (d1.cell_rank == 0).all()
    d2 = decompose(m81, 2)
    assert sorted(np.bincount(d2.cell_rank).tolist()) == [40, 41]
    m9 = CartesianMesh(3, 2, True)
    d3 = decompose(m9, 3)
    assert np.bincount(d3.cell_rank).tolist() == [3, 3, 3]
    faces, _ = interior_faces(m9)
    brute = {i for i, (a, b) in enumerate(faces) if d3.cell_rank[a] != d3.cell_rank[b]}
    got = set()
    for r1 in range(3):
        for r2 in range(r1 + 1, 3):
            got |= set(boundary_face_order(m9, d3, (r1, r2)).tolist())
    assert got == brute
    assert boundary_face_order(m81, d1, (0, 0)).size == 0
    with pytest.raises(ConfigError):
        decompose(m9, 0)
    with pytest.raises(ConfigError):
        decompose(m9, 10)
    with pytest.raises(ConfigError):
        boundary_face_order(m9, d3, (0, 3))


def _payload(plan, peer, nvar=4):
    import torch
    # row = (face index, local cell, side) -- what the sender holds for that face
    f = torch.from_numpy(plan.faces[peer]).double()
    c = torch.from_numpy(plan.local_cell[peer]).double()
    s = torch.from_numpy(plan.local_side[peer].astype(np.float64))
    return torch.stack([f * 1000 + c + 0.5 * s + v for v in range(nvar)], dim=1)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    from paper_1806_07984_b200.decomposition import exchange_traces, global_dt
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mesh = AdaptiveMesh([(2, (i, j)) for i in range(9) for j in range(9)], 2, True)
    dec = decompose(mesh, world)
    plan = exchange_plan(mesh, dec, rank)
    recv = exchange_traces(dist, plan, {p: _payload(plan, p) for p in plan.peers})
    ok = True
    for p in plan.peers:
        peer_plan = exchange_plan(mesh, dec, p)
        ok &= bool(np.array_equal(peer_plan.faces[rank], plan.faces[p]))
        ok &= bool(torch.equal(recv[p], _payload(peer_plan, rank)))
    dt = global_dt(dist, 0.1 * (rank + 1), cfl=0.5)
    quiet = global_dt(dist, None if rank == 1 else 0.3)       # a rank without a positive speed
    try:
        global_dt(dist, None)
        none_raises = False
    except Exception as e:  # EnclaveDgError on every rank
        none_raises = type(e).__name__ == "EnclaveDgError"
    ok &= quiet == 0.3 and none_raises
    q.put((rank, ok, len(plan.peers), float(dt)))
    dist.destroy_process_group()


def test_exchange_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get() for _ in range(2))
    assert [r[1] for r in res] == [True, True]
    assert [r[2] for r in res] == [1, 1]
    assert [r[3] for r in res] == [0.5 * 0.1, 0.5 * 0.1]


@pytest.mark.gpu
@pytest.mark.parametrize("dim,m,n", [(2, 4, 4), (3, 5, 5)])
def test_gpu_pack_unpack_bit_exact(dim, m, n):
    """edg_pack_face_traces / edg_unpack_face_traces against plain indexing
    (a copy: bit-exact), on the 3-rank exchange plan of a uniform mesh."""
    import torch
    from paper_1806_07984_b200.decomposition import pack_boundary_traces, unpack_boundary_traces
    mesh = CartesianMesh(9 if dim == 2 else 6, dim, True)
    dec = decompose(mesh, 3)
    g = torch.Generator(device="cuda").manual_seed(7)
    shape = (mesh.ncells, 2 * dim, m, n ** (dim - 1))
    tq = torch.rand(shape, dtype=torch.float64, device="cuda", generator=g)
    tf = torch.rand(shape, dtype=torch.float64, device="cuda", generator=g)
    for rank in range(3):
        plan = exchange_plan(mesh, dec, rank)
        assert plan.peers
        for p in plan.peers:
            c = torch.from_numpy(plan.local_cell[p]).cuda()
            s = torch.from_numpy(plan.local_fs[p].astype(np.int64)).cuda()
            want = torch.stack([tq[c, s].flatten(1), tf[c, s].flatten(1)], dim=1)
            got = pack_boundary_traces(plan, p, tq, tf)
            torch.cuda.synchronize()
            assert torch.equal(got, want)
            k = got.shape[0]
            slots = np.random.default_rng(rank).permutation(k + 3)[:k]
            ghost = torch.zeros((k + 3, 2, got.shape[-1]), dtype=torch.float64, device="cuda")
            unpack_boundary_traces(got, slots, ghost)
            torch.cuda.synchronize()
            assert torch.equal(ghost[torch.from_numpy(slots.astype(np.int64)).cuda()], got)
    # the face side each rank packs is the side that touches the peer cell
    plan = exchange_plan(mesh, dec, 0)
    faces, keys = interior_faces(mesh)
    for p in plan.peers:
        for f, c, fs in zip(plan.faces[p], plan.local_cell[p], plan.local_fs[p]):
            other = faces[f, 1] if faces[f, 0] == c else faces[f, 0]
            assert mesh.nbr[c, fs] == other


@pytest.mark.gpu
@pytest.mark.parametrize("R", [2, 3])
def test_gpu_redundant_riemann_agreement(R):
    """SPEC.md rank-sim invariants on the device path: after the predictor,
    packing each rank's own traces and swapping the buffers, the Rusanov
    outcome each rank computes for a shared face is bitwise equal to its
    peer's and to the single-domain outcome (rank-count transparency at the
    face level)."""
    import torch
    import paper_1806_07984_b200 as edg
    from paper_1806_07984_b200.decomposition import pack_boundary_traces
    mesh = CartesianMesh(9, 2, True)
    pde, p = edg.pde.euler(2), 3
    b = edg.basis.get_basis(p)
    n = p + 1
    rng = np.random.default_rng(11)
    Q = np.empty((mesh.ncells, 4, n, n))
    Q[:, 0] = 1.0 + 0.1 * rng.random((mesh.ncells, n, n))
    Q[:, 1] = 0.2 * rng.standard_normal((mesh.ncells, n, n))
    Q[:, 2] = 0.2 * rng.standard_normal((mesh.ncells, n, n))
    Q[:, 3] = 2.5 + 0.1 * rng.random((mesh.ncells, n, n))
    h = 1.0 / 9
    out = edg.kernels.stp_picard_batch(torch.from_numpy(Q).cuda(), pde, 0.2 * h / 7, b, (h, h))
    tq, tf = out["trace_q"], out["trace_f"]
    dec = decompose(mesh, R)
    faces, keys = interior_faces(mesh)
    axis = np.array([k[0] for k in keys])
    plans = [exchange_plan(mesh, dec, r) for r in range(R)]
    sent = {(r, q): pack_boundary_traces(plans[r], q, tq, tf) for r in range(R) for q in plans[r].peers}
    outcome = {}
    for r in range(R):
        for q in plans[r].peers:
            own, recv = sent[(r, q)][:, 0], sent[(q, r)][:, 0]          # trace_q rows (k, m*n)
            lo_mine = torch.from_numpy(plans[r].local_side[q] == 0).cuda()[:, None]
            lo, hi = torch.where(lo_mine, own, recv), torch.where(lo_mine, recv, own)
            res = torch.empty_like(lo)
            ax = axis[plans[r].faces[q]]
            for a in range(2):
                sel = torch.from_numpy(np.nonzero(ax == a)[0]).cuda()
                res[sel] = edg.kernels.riemann_rusanov_batch(lo[sel].reshape(-1, 4, n).contiguous(),
                                                             hi[sel].reshape(-1, 4, n).contiguous(),
                                                             pde, a).reshape(-1, 4 * n)
            outcome[(r, q)] = res
            # single-domain reference for the same faces
            f = plans[r].faces[q]
            for a in range(2):
                fa = f[ax == a]
                if fa.size == 0:
                    continue
                lo1 = tq[torch.from_numpy(faces[fa, 0]).cuda(), 2 * a + 1].contiguous()
                hi1 = tq[torch.from_numpy(faces[fa, 1]).cuda(), 2 * a].contiguous()
                want = edg.kernels.riemann_rusanov_batch(lo1, hi1, pde, a).reshape(-1, 4 * n)
                assert torch.equal(res[torch.from_numpy(np.nonzero(ax == a)[0]).cuda()], want)
    for r in range(R):
        for q in plans[r].peers:
            assert torch.equal(outcome[(r, q)], outcome[(q, r)])


@pytest.mark.gpu
@pytest.mark.parametrize("R", [2, 3])
def test_gpu_sharded_step_equals_single_domain(R):
    """A whole DG step assembled rank by rank -- predictor traces packed and
    swapped between ranks, each rank's face solves from its own and the
    received traces, the generic corrector on each rank's cells -- is
    bitwise the R = 1 run through the same kernels (SPEC.md rank-sim "R=2
    ... Q_h bitwise equal to R=1 run"), and that run matches the fused
    single-domain solver step to 1e-13 relative.  Ranks run one after
    another on one GPU; no rank's kernel waits on another's."""
    import torch
    import paper_1806_07984_b200 as edg
    from paper_1806_07984_b200.decomposition import pack_boundary_traces
    N = 9
    cfg = edg.configs.CONFIGS["cfg2"].with_(cells=N)
    mesh = CartesianMesh(N, 2, True, extent=N / 243)
    s = edg.solver.DGSolver(edg.pde.euler(2), cfg.order, mesh, cfg.cfl)
    s.set_state(edg.configs.initial_dg_uniform(edg.configs.CONFIGS["cfg2"], window=(100, N)))
    s.step()
    torch.cuda.synchronize()
    q_single = s.state().clone()
    tq, tf = s.trace_q, s.trace_f
    C_, m = mesh.ncells, tq.shape[2]
    faces, keys = interior_faces(mesh)
    axis = np.array([k[0] for k in keys])
    F_ = faces.shape[0]
    assert F_ == 2 * C_                                  # periodic: face a*C + c has lo cell c
    side_face = np.empty((C_, 4), dtype=np.int32)
    for a in range(2):
        side_face[:, 2 * a + 1] = a * C_ + np.arange(C_)
        side_face[:, 2 * a] = a * C_ + mesh.nbr[:, 2 * a]
    side_face = torch.from_numpy(side_face).cuda()
    # R = 1 through the same face-solve + generic-corrector kernels
    oc1 = torch.empty((F_,) + tuple(tq.shape[2:]), dtype=torch.float64, device="cuda")
    for a in range(2):
        fa = np.nonzero(axis == a)[0]
        oc1[torch.from_numpy(fa).cuda()] = edg.kernels.riemann_rusanov_batch(
            tq[torch.from_numpy(faces[fa, 0]).cuda(), 2 * a + 1].contiguous(),
            tq[torch.from_numpy(faces[fa, 1]).cuda(), 2 * a].contiguous(), s.pde, a)
    q_r1 = edg.kernels.corrector_batch(s.pde, s.basis, s.q_end, tf, (1 / 243,) * 2, outcomes=oc1,
                                       side_face=side_face).reshape(q_single.shape)
    rel = float(((q_r1 - q_single).abs().max() / q_single.abs().max()).item())
    print(f"generic-table corrector vs fused grid solver step: rel L-inf {rel:.3e}")
    assert rel <= 1e-13
    dec = decompose(mesh, R)
    plans = [exchange_plan(mesh, dec, r) for r in range(R)]
    sent = {(r, q): pack_boundary_traces(plans[r], q, tq, tf) for r in range(R) for q in plans[r].peers}
    q_sharded = torch.full_like(q_single, float("nan"))
    for r in range(R):
        oc = torch.zeros((F_,) + tuple(tq.shape[2:]), dtype=torch.float64, device="cuda")
        mine = dec.cell_rank[faces] == r
        inner = np.nonzero(mine.all(axis=1))[0]
        for a in range(2):
            fa = inner[axis[inner] == a]
            lo = tq[torch.from_numpy(faces[fa, 0]).cuda(), 2 * a + 1].contiguous()
            hi = tq[torch.from_numpy(faces[fa, 1]).cuda(), 2 * a].contiguous()
            oc[torch.from_numpy(fa).cuda()] = edg.kernels.riemann_rusanov_batch(lo, hi, s.pde, a)
        for q in plans[r].peers:
            own, recv = sent[(r, q)][:, 0], sent[(q, r)][:, 0]
            lo_mine = torch.from_numpy(plans[r].local_side[q] == 0).cuda()[:, None]
            lo, hi = torch.where(lo_mine, own, recv), torch.where(lo_mine, recv, own)
            f = plans[r].faces[q]
            for a in range(2):
                sel = np.nonzero(axis[f] == a)[0]
                if sel.size == 0:
                    continue
                st = torch.from_numpy(sel).cuda()
                oc[torch.from_numpy(f[sel]).cuda()] = edg.kernels.riemann_rusanov_batch(
                    lo[st].reshape((-1,) + tuple(tq.shape[2:])).contiguous(),
                    hi[st].reshape((-1,) + tuple(tq.shape[2:])).contiguous(), s.pde, a)
        out = edg.kernels.corrector_batch(s.pde, s.basis, s.q_end, tf, (1 / 243,) * 2, outcomes=oc,
                                          side_face=side_face)
        cells = torch.from_numpy(dec.cells_of(r).astype(np.int64)).cuda()
        q_sharded[cells] = out.reshape(q_single.shape)[cells]
    torch.cuda.synchronize()
    assert torch.equal(q_sharded, q_r1)              # rank-count transparency, bitwise


def test_adaptive_plan_carries_the_chain_paths():
    """A rank-boundary hanging face carries the leaf's interpolation path in the
    plan, identical on both ranks (the receiver of a coarse owner's trace
    evaluates it at the leaf's points)."""
    G = GOLDEN["refined"]
    cells = [_key(c) for c in G["cells"]]
    mesh = AdaptiveMesh(cells, 2, True)
    for R in (2, 3, 4):
        dec = decompose(mesh, R)
        plans = [exchange_plan(mesh, dec, r) for r in range(R)]
        hanging = 0
        for p in plans:
            for q in p.peers:
                assert np.array_equal(p.vpath[q], plans[q].vpath[p.rank])
                assert np.array_equal(p.vdepth[q], plans[q].vdepth[p.rank])
                hanging += int((p.vdepth[q] > 0).sum())
        assert hanging > 0
