"""Full-size, full-length parity of the GPU path against the CPU oracle.

    python tools/parity_report.py [--configs cfg1,cfg2,...] [--procs N] [--out profiles/parity_round1.json]

Runs every BASELINE configuration at its stated size for its stated number
of steps on the GPU (solver.DGSolver / FVSolver, CUDA-graph path) and with
the batched oracle (oracle/batched.py, bit-equal up to ULPs to the reference
kernels; the predictor is farmed out to N worker processes), and records the
relative L-infinity error of the final state, the dt histories and the
Picard-count histogram.  For the stated CFL of config 2, which the reference
scheme itself does not survive (hard part 1), it also
records the first non-finite step and the error up to it, and runs the
parity-safe variant (CFL 0.2).  Test infrastructure: it imports oracle/.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

from paper_1806_07984_b200 import configs as cf  # noqa: E402

_W = {}


def _pde(name, dim, velocity):
    from oracle import ops
    return ops.advection(velocity, dim) if name == "advection" else ops.make_pde(name, dim=dim)


def _init_worker(name, dim, velocity, order):
    from oracle import ops
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    _W["pde"] = _pde(name, dim, velocity)
    _W["basis"] = ops.basis_for(order)


def _stp_chunk(args):
    from oracle import batched
    Q, dt, edges = args
    return batched.predictor_picard_b(Q, _W["pde"], dt, _W["basis"], edges)


def _stp_cell(args):
    from oracle import ops
    q, dt, edges = args
    return ops.predictor_picard(q, _W["pde"], dt, _W["basis"], edges)


def _fv_chunk(args):
    from oracle import batched
    P, dt, edges, halos = args
    return batched.fv_update_b(P, _W["pde"], dt, edges, halos)


def rel(a, b):
    den = np.abs(b).max()
    return float(np.abs(a - b).max() / (den if den > 0 else 1.0))


def oracle_uniform_step(pool, cfg, Q, nchunks):
    """One Algorithm-1 step of the batched oracle, predictor in the pool."""
    from oracle import batched, drivers, ops
    pde = _pde(cfg.pde, cfg.dim, cfg.velocity)
    basis = ops.basis_for(cfg.order)
    N, d = cfg.cells, cfg.dim
    h = 1.0 / N
    dt = batched.stable_dt_b(Q, h, pde, cfg.order, cfg.cfl, d)
    parts = pool.map(_stp_chunk, [(c, dt, (h,) * d) for c in np.array_split(Q, nchunks)])
    st = {k: np.concatenate([p[k] for p in parts]) for k in ("q_end", "iterations")}
    for fam in ("trace_q", "trace_f"):
        st[fam] = {key: np.concatenate([p[fam][key] for p in parts]) for key in parts[0][fam]}
    outc = drivers.uniform_outcomes(st["trace_q"], pde, N, d, cfg.periodic)
    return batched.correct_b(st["q_end"], st["trace_f"], outc, basis, (h,) * d), dt, st["iterations"]


def run_uniform(pool, name, cfg, nchunks, lockstep=False):
    """GPU and oracle from the same initial state for the stated steps; with
    lockstep=True the two are compared after every step."""
    import torch
    from paper_1806_07984_b200 import mesh as M, pde as P, solver as S
    t0 = time.time()
    Q0 = cf.initial_dg_uniform(cfg)
    pde = P.advection(cfg.velocity) if cfg.pde == "advection" else P.euler(cfg.dim)
    s = S.DGSolver(pde, cfg.order, M.CartesianMesh(cfg.cells, cfg.dim, cfg.periodic), cfg.cfl, check_finite=False)
    s.set_state(Q0)
    res = {"config": name, "cells": int(Q0.shape[0]), "steps": cfg.steps, "cfl_safety": cfg.cfl}
    Q = Q0.copy()
    dts, its, errs = [], None, []
    if not lockstep:
        s.run(cfg.steps, graph=True)
        for _ in range(cfg.steps):
            Q, dt, its = oracle_uniform_step(pool, cfg, Q, nchunks)
            dts.append(dt)
    else:
        for k in range(cfg.steps):
            s.step()
            Q, dt, its = oracle_uniform_step(pool, cfg, Q, nchunks)
            dts.append(dt)
            G = s.state().cpu().numpy()
            if not (np.isfinite(G).all() and np.isfinite(Q).all()):
                res.setdefault("first_nonfinite_step", k + 1)
                res["gpu_finite_at_first_nonfinite"] = bool(np.isfinite(G).all())
                res["oracle_finite_at_first_nonfinite"] = bool(np.isfinite(Q).all())
                break
            errs.append(rel(G, Q))
        res["rel_linf_per_step_until_nonfinite"] = errs
    torch.cuda.synchronize()
    Qg = s.state().cpu().numpy()
    dtg = s.dt_history()[:len(dts)]
    res.update({"rel_linf_final": rel(Qg, Q), "finite_gpu": bool(np.isfinite(Qg).all()),
                "finite_oracle": bool(np.isfinite(Q).all()),
                "dt_rel_max": rel(dtg, np.array(dts)) if np.isfinite(dts).all() else None,
                "picard_last_step_equal": bool(np.array_equal(s.iterations.cpu().numpy(), its)),
                "picard_hist_last_step": {int(k): int(v) for k, v in zip(*np.unique(its, return_counts=True))},
                "within_1e-10": bool(rel(Qg, Q) <= 1e-10), "wall_s": time.time() - t0})
    return res


def run_fv(pool, cfg, nchunks):
    import torch
    from oracle import batched, drivers
    from paper_1806_07984_b200 import pde as P, solver as S
    P0 = cf.initial_fv(cfg)
    s = S.FVSolver(P.euler(3), cfg.cells, cfg.patch, cfg.cfl)
    s.set_state(P0)
    s.run(cfg.steps, graph=True)
    torch.cuda.synchronize()
    Pg = s.state().cpu().numpy()
    pde = _pde("euler", 3, ())
    Pq = P0.copy()
    h = 1.0 / cfg.cells
    edges = (h * cfg.patch,) * 3
    dts = []
    for _ in range(cfg.steps):
        dt = drivers.fv_dt(Pq, pde, cfg.cfl, h)
        halos = drivers.fv_halos(Pq)
        idx = np.array_split(np.arange(Pq.shape[0]), nchunks)
        parts = pool.map(_fv_chunk, [(Pq[i], dt, edges, {k: v[i] for k, v in halos.items()}) for i in idx])
        Pq = np.concatenate(parts)
        dts.append(dt)
    return {"config": "cfg4", "cells": cfg.cells ** 3, "steps": cfg.steps, "cfl_safety": cfg.cfl,
            "bitwise_equal": bool(np.array_equal(Pg, Pq)), "rel_linf_final": rel(Pg, Pq),
            "dt_bitwise_equal": bool(np.array_equal(s.dt_history(), np.array(dts))),
            "within_1e-10": bool(rel(Pg, Pq) <= 1e-10)}


def run_amr(pool, cfg):
    import torch
    from oracle import ops, spacetree, transfer
    from paper_1806_07984_b200 import mesh as M, pde as P, solver as S
    cells = cf.amr_cells(cfg)
    mesh = M.AdaptiveMesh(cells, 2, True)
    s = S.DGSolver(P.euler(2), cfg.order, mesh, cfg.cfl)
    Q0 = cf.initial_dg_amr(cfg, mesh.cells)
    s.set_state(Q0)
    s.run(cfg.steps, graph=True)
    torch.cuda.synchronize()
    Qg = s.state().cpu().numpy()
    forest = spacetree.FaceForest(cells, 2, True)
    pde = _pde("euler", 2, ())
    basis = ops.basis_for(cfg.order)
    ops_t = transfer.transfer_for(cfg.order)
    Q = {k: Q0[i] for i, k in enumerate(forest.sfc)}
    dts = []
    for step in range(cfg.steps):
        dt = ops.stable_dt(((min(forest.cell_edges(k[0])), Q[k]) for k in forest.sfc), pde, cfg.order, cfg.cfl, 2)
        stl = pool.map(_stp_cell, [(Q[k], dt, forest.cell_edges(k[0])) for k in forest.sfc], chunksize=256)
        stores = dict(zip(forest.sfc, stl))
        outcome, acc = {}, {}
        for f in forest.leaf_faces():
            a = f.axis
            tr = [None, None]
            for sd in (0, 1):
                if f.sides[sd] == "cell":
                    tr[sd] = stores[f.owners[sd]].trace_q[(a, 1 - sd)]
                elif f.sides[sd] == "virtual":
                    tr[sd] = transfer.to_virtual(ops_t, stores[f.owners[sd]].trace_q[(a, 1 - sd)], f.child_pos)
            tr[0] = tr[1] if f.sides[0] == "boundary" else tr[0]
            tr[1] = tr[0] if f.sides[1] == "boundary" else tr[1]
            out = ops.rusanov(tr[0], tr[1], pde, a)
            if f.parent is not None:
                buf = acc.setdefault(f.parent.key, transfer.ParentAccumulator())
                transfer.accumulate_restriction(ops_t, buf, out, f.child_pos, step)
            outcome[f.key] = out
        for key, buf in acc.items():
            outcome[key] = buf.outcome
        Q = {k: ops.correct(stores[k], {(a, sd): outcome[forest.side_face_key(k, a, sd)]
                                        for a in range(2) for sd in (0, 1)}, basis, forest.cell_edges(k[0]))
             for k in forest.sfc}
        dts.append(dt)
    Qo = np.stack([Q[k] for k in forest.sfc])
    return {"config": "cfg5", "cells": len(cells), "steps": cfg.steps, "cfl_safety": cfg.cfl,
            "rel_linf_final": rel(Qg, Qo), "dt_rel_max": rel(s.dt_history(), np.array(dts)),
            "within_1e-10": bool(rel(Qg, Qo) <= 1e-10)}


def main():
    import multiprocessing as mp
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="cfg1,cfg2s,cfg2,cfg3,cfg4,cfg5")
    ap.add_argument("--procs", type=int, default=os.cpu_count() or 4)
    ap.add_argument("--out", default=os.path.join(REPO, "gpurun_out", "parity.json"))
    a = ap.parse_args()
    report = {"procs": a.procs, "results": []}
    ctx = mp.get_context("fork")
    for name in a.configs.split(","):
        base = "cfg2" if name == "cfg2s" else name
        cfg = cf.CONFIGS[base].with_(cfl=0.2) if name == "cfg2s" else cf.CONFIGS[base]
        init = (cfg.pde, cfg.dim, cfg.velocity, max(cfg.order, 1))
        t = time.time()
        with ctx.Pool(a.procs, initializer=_init_worker, initargs=init) as pool:
            if cfg.kind == "fv":
                r = run_fv(pool, cfg, 4 * a.procs)
            elif cfg.kind == "dg-amr":
                r = run_amr(pool, cfg)
            else:
                r = run_uniform(pool, name, cfg, 4 * a.procs, lockstep=(name == "cfg2"))
        r["wall_s"] = time.time() - t
        report["results"].append(r)
        print(json.dumps(r), flush=True)
        json.dump(report, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
