"""The N > 1 plumbing of bench.py on CPU with the gloo backend, world size 2:
replicas are timed as the max over ranks, the reference arm runs on rank 0
only.  (The hot path itself does not shard in this tier: DESIGN.md section 7.)"""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import bench
    ws, r, _ = bench.dist_env()
    dist = bench.dist_init(ws, "gloo")
    got = bench.max_over_ranks(dist, 10.0 * (r + 1), "cpu")
    dist.barrier()
    q.put((r, got))
    dist.destroy_process_group()


def test_max_over_ranks_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = dict(q.get() for _ in range(2))
    assert res == {0: 20.0, 1: 20.0}


def test_reference_arm_nonzero_rank_does_no_work(monkeypatch, capsys):
    import bench
    monkeypatch.setenv("RANK", "1")
    monkeypatch.setenv("WORLD_SIZE", "2")
    args = type("A", (), dict(steps=1, warmup=0, cfl=None, gpus=2))()
    bench.run_reference(args, bench.cf.CONFIGS["cfg1"])
    assert capsys.readouterr().out == ""
