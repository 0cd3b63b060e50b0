"""The sharded step (row f3; SPEC.md:425-508 rank-sim).

CPU: the host layout of every rank (local / ghost numbering, neighbour
tables, send / receive rows in boundary_face_order) is checked by exchanging
identifier rows -- after pack -> exchange -> unpack, every side a local cell's
face solve reads must hold the right global neighbour's trace -- both in one
process and through torch.distributed (gloo, world size 2).
GPU (marked): R = 2, 3 ranks emulated in one process (SPEC.md:500
"interleaved" mode; the ranks' kernels never wait on one another) are
bitwise the single-domain DGSolver run over 5 steps; the torch.distributed
step path (two priority streams) is bitwise too, with NCCL at world size 1
and with two real ranks over gloo (host-staged exchange: neither rank's
device work ever waits on the other's, so the two processes can share the
one GPU).
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1806_07984_b200.decomposition import decompose
from paper_1806_07984_b200.mesh import CartesianMesh
from paper_1806_07984_b200.sharded import shard_layout


def _ids(mesh, lay):
    """Trace rows of one rank filled with global ids: row (cell, side) = cell * 2d + side."""
    d2 = 2 * mesh.dim
    L, G = lay.local.size, lay.ghost.size
    rows = np.full((L + G) * d2, -1, dtype=np.int64)
    rows[:L * d2] = (lay.local[:, None] * d2 + np.arange(d2)[None, :]).ravel()
    return rows


def _check_rank(mesh, lay, rows):
    d2 = 2 * mesh.dim
    for i, c in enumerate(lay.local):
        for fs in range(d2):
            g = mesh.nbr[c, fs]
            nb = lay.nbr[i, fs]
            if g < 0:
                assert nb == -1
                continue
            assert nb >= 0
            # the face solve of (cell, side fs) reads the neighbour's trace on side fs ^ 1
            assert rows[nb * d2 + (fs ^ 1)] == g * d2 + (fs ^ 1), (lay.rank, c, fs)
    remote = [i for i in range(lay.local.size) if (lay.nbr[i] >= lay.local.size).any()]
    assert sorted(lay.skeleton.tolist()) == remote
    assert sorted(lay.skeleton.tolist() + lay.enclave.tolist()) == list(range(lay.local.size))


@pytest.mark.parametrize("N,dim,periodic", [(9, 2, True), (4, 2, True), (6, 3, False), (3, 3, True)])
@pytest.mark.parametrize("R", [2, 3, 5])
def test_layout_identifier_exchange(N, dim, periodic, R):
    mesh = CartesianMesh(N, dim, periodic)
    dec = decompose(mesh, R)
    lays = [shard_layout(mesh, dec, r) for r in range(R)]
    rows = [_ids(mesh, l) for l in lays]
    send = {(l.rank, q): rows[l.rank][l.send_rows[q]] for l in lays for q in l.peers}
    for l in lays:
        for q in l.peers:
            assert lays[q].send_rows[l.rank].size == l.recv_rows[q].size
            rows[l.rank][l.recv_rows[q]] = send[(q, l.rank)]
    for l in lays:
        _check_rank(mesh, l, rows[l.rank])
    assert sum(l.local.size for l in lays) == mesh.ncells


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    from paper_1806_07984_b200.sharded import TorchComm
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mesh = CartesianMesh(9, 2, True)
    dec = decompose(mesh, world)
    lay = shard_layout(mesh, dec, rank)
    rows = torch.from_numpy(_ids(mesh, lay).astype(np.float64))
    comm = TorchComm(dist)
    send = {p: rows[torch.from_numpy(lay.send_rows[p])].reshape(-1, 1).clone() for p in lay.peers}
    recv = {p: torch.empty_like(send[p]) for p in lay.peers}
    comm.exchange(rank, send, recv)
    for p in lay.peers:
        rows[torch.from_numpy(lay.recv_rows[p])] = recv[p].reshape(-1)
    ok = True
    try:
        _check_rank(mesh, lay, rows.numpy().astype(np.int64))
    except AssertionError:
        ok = False
    slots = torch.full((4,), 2 ** 63 - 1, dtype=torch.int64)
    if rank == 1:
        slots[2] = 12345
    comm.allreduce_min_(slots)
    ok &= slots.tolist() == [2 ** 63 - 1, 2 ** 63 - 1, 12345, 2 ** 63 - 1]
    q.put((rank, ok))
    dist.destroy_process_group()


def test_layout_exchange_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert sorted(q.get() for _ in range(2)) == [(0, True), (1, True)]


# ---------------------------------------------------------------- GPU --

def _single(edg, cfg, N, Q0, steps):
    import torch
    pde = edg.pde.make_pde(cfg.pde, dim=cfg.dim)
    s = edg.solver.DGSolver(pde, cfg.order, CartesianMesh(N, cfg.dim, cfg.periodic), cfg.cfl)
    s.set_state(Q0)
    s.run(steps, graph=False)
    torch.cuda.synchronize()
    return s.state().cpu().numpy(), s.dt_history()


@pytest.mark.gpu
@pytest.mark.parametrize("name,N", [("cfg2", 27), ("cfg3", 9)])
@pytest.mark.parametrize("R", [2, 3])
def test_gpu_emulated_ranks_bitwise(name, N, R):
    import torch
    import paper_1806_07984_b200 as edg
    cfg = edg.configs.CONFIGS[name].with_(cells=N, cfl=0.2)
    Q0 = edg.configs.initial_dg_uniform(cfg)
    steps = 5
    ref, ref_dt = _single(edg, cfg, N, Q0, steps)
    mesh = CartesianMesh(N, cfg.dim, cfg.periodic)
    dec = decompose(mesh, R)
    pde = edg.pde.make_pde(cfg.pde, dim=cfg.dim)
    ranks = [edg.sharded.ShardedDGSolver(pde, cfg.order, mesh, cfg.cfl, dec, r) for r in range(R)]
    for r in ranks:
        r.set_state(Q0)
    for _ in range(steps):
        edg.sharded.ShardedDGSolver.emulate_step(ranks)
    out = torch.zeros((mesh.ncells,) + tuple(ranks[0].Q.shape[1:]), dtype=torch.float64, device="cuda")
    for r in ranks:
        r.gather_into(out)
        r.check_status()
        assert np.array_equal(r.dt_history(), ref_dt)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), ref)


@pytest.mark.gpu
def test_gpu_torch_distributed_step_world1():
    """The step() path (priority streams, TorchComm over NCCL) with one rank."""
    import torch
    import torch.distributed as dist
    import paper_1806_07984_b200 as edg
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        cfg = edg.configs.CONFIGS["cfg2"].with_(cells=27, cfl=0.2)
        Q0 = edg.configs.initial_dg_uniform(cfg)
        ref, _ = _single(edg, cfg, 27, Q0, 4)
        mesh = CartesianMesh(27, 2, True)
        s = edg.sharded.ShardedDGSolver(edg.pde.euler(2), cfg.order, mesh, cfg.cfl, decompose(mesh, 1), 0,
                                        comm=edg.sharded.TorchComm(dist))
        s.set_state(Q0)
        for _ in range(4):
            s.step()
        torch.cuda.synchronize()
        assert np.array_equal(s.state().cpu().numpy(), ref)
    finally:
        dist.destroy_process_group()


def _gpu_worker(rank, world, port, q, N):
    """One rank of a real torch.distributed sharded run (gloo: host-staged
    exchange, so no device work of one rank ever waits on the other's)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    import paper_1806_07984_b200 as edg
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = edg.configs.CONFIGS["cfg2"].with_(cells=N, cfl=0.2)
        mesh = CartesianMesh(N, 2, True)
        s = edg.sharded.ShardedDGSolver(edg.pde.euler(2), cfg.order, mesh, cfg.cfl, decompose(mesh, world), rank,
                                        comm=edg.sharded.TorchComm(dist))
        s.set_state(edg.configs.initial_dg_uniform(cfg))
        for _ in range(3):
            s.step()
        torch.cuda.synchronize()
        s.check_status()
        q.put((rank, s.layout.local, s.state().cpu().numpy(), s.dt_history()))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_gpu_torch_distributed_world2_bitwise():
    """Two ranks through the torch.distributed step path (priority streams,
    per-neighbour exchange, dt slots all-reduced) reproduce the single-domain
    run bitwise."""
    import torch
    import paper_1806_07984_b200 as edg
    N = 27
    cfg = edg.configs.CONFIGS["cfg2"].with_(cells=N, cfl=0.2)
    ref, ref_dt = _single(edg, cfg, N, edg.configs.initial_dg_uniform(cfg), 3)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, 2, port, q, N)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]     # before join: the payloads exceed the pipe buffer
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    out = np.empty_like(ref)
    for rank, local, Q, dt in res:
        out[local] = Q
        assert np.array_equal(dt, ref_dt)
    assert np.array_equal(out, ref)
