"""Full-size, full-length parity fixtures from the pinned CPU oracle.

    python tests/golden/make_full_parity.py [--configs cfg2s,cfg2,cfg3,cfg4,cfg5] [--procs N]

Runs every BASELINE configuration at its stated size for its stated number
of steps with the batched oracle (oracle/fullrun.py: oracle/batched.py for the
uniform grids and FV, the per-cell oracle/ops.py on the adaptive mesh; the
oracle is pinned to the reference package by tests/golden/make_golden.py and
tests/test_oracle_golden.py) and writes compact fixtures the GPU tests
(`tests/test_gpu_fullsize.py`) compare the device path against:

* per step: dt, the Picard-count histogram, the conserved integrals
  (sum over cells of volume x quadrature-weighted DoFs, per component);
* final state: the full (m, n^d) blocks of 1024 seeded sample cells, and for
  EVERY cell a fingerprint f_c = sum(r * Q_c) with seeded weights r in
  [0.5, 1.5) (oracle/fullrun.py), so a deviation anywhere shows up;
* cfg4 (FV, bitwise on the GPU): SHA-256 of the final state bytes and of the
  dt history, plus 1024 seeded sample volumes;
* cfg2 at the stated CFL 0.9/(2p+1), which the reference scheme itself does
  not survive: the sample cells after each of steps 1-5 and the first step
  whose state is non-finite;
* cfg3 (the bench workload): for each of its 20 steps, the input state of up
  to two cells per Picard count that occurs in that step (`refarm_cfg3.npz`),
  which bench.py's reference arm times the reference kernels on.

Test infrastructure: imports oracle/.  Takes about an hour on 8 cores (cfg3
dominates).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

from oracle import fullrun, ops, spacetree  # noqa: E402
from paper_1806_07984_b200 import configs as cf  # noqa: E402

SAMPLE = 1024
SAMPLE_SEED = 1234
FP_SEED = 4321


def cfg_of(name):
    if name == "cfg2s":
        return cf.CONFIGS["cfg2"].with_(cfl=0.2)
    return cf.CONFIGS[name]


def sample_cells(C):
    return np.sort(np.random.default_rng(SAMPLE_SEED).choice(C, size=min(SAMPLE, C), replace=False))


def dg_run(name, procs, out):
    cfg = cfg_of(name)
    t0 = time.time()
    basis = ops.basis_for(cfg.order)
    wnd = fullrun.tensor_weights(basis.weights, cfg.dim)
    amr = cfg.kind == "dg-amr"
    if amr:
        cells = cf.amr_cells(cfg)
        forest = spacetree.FaceForest(cells, cfg.dim, cfg.periodic)
        Q = cf.initial_dg_amr(cfg, forest.sfc)
        vol = np.array([np.prod(forest.cell_edges(k[0])) for k in forest.sfc])
    else:
        Q = cf.initial_dg_uniform(cfg)
        vol = (1.0 / cfg.cells) ** cfg.dim
    C = Q.shape[0]
    sample = sample_cells(C)
    r = fullrun.fingerprint_weights(FP_SEED, Q.shape[1:])
    nmax = 2 * cfg.n
    stated09 = name == "cfg2"
    steps = cfg.steps
    rec = {"dt": [], "hist": [], "integrals": [fullrun.integrals(Q, wnd, vol)]}
    early = []          # cfg2 at 0.9: sample states after steps 1..5
    strata_q, strata_step, strata_its = [], [], []
    first_nonfinite = 0
    nchunks = 4 * procs
    with fullrun.pool_for(cfg, procs) as pool:
        for k in range(steps):
            Qin = Q
            if amr:
                Q, dt, its = fullrun.amr_step(pool, cfg, forest, Q, k)
            else:
                Q, dt, its = fullrun.uniform_step(pool, cfg, Q, nchunks)
            rec["dt"].append(dt)
            rec["hist"].append(np.bincount(its, minlength=nmax + 1)[:nmax + 1])
            rec["integrals"].append(fullrun.integrals(Q, wnd, vol))
            if name == "cfg3":
                rng = np.random.default_rng(100 + k)
                for v in np.unique(its):
                    idx = np.flatnonzero(its == v)
                    for c in rng.choice(idx, size=min(2, idx.size), replace=False):
                        strata_q.append(Qin[c])
                        strata_step.append(k + 1)
                        strata_its.append(v)
            if stated09 and k < 5:
                early.append(Q[sample].copy())
            fin = bool(np.isfinite(Q).all())
            print(f"{name} step {k + 1}/{steps} dt={dt:.6e} mean_it={its.mean():.3f} finite={fin} "
                  f"t={time.time() - t0:.0f}s", flush=True)
            if not fin:
                first_nonfinite = k + 1
                break
    fix = {"config": name, "cells": C, "steps_run": len(rec["dt"]), "cfl": cfg.cfl,
           "dt": np.array(rec["dt"]), "hist": np.array(rec["hist"]), "integrals": np.array(rec["integrals"]),
           "sample": sample, "fp_seed": FP_SEED, "first_nonfinite_step": first_nonfinite}
    if stated09:
        fix["early_states"] = np.array(early)
    else:
        fix["final_sample"] = Q[sample]
        fix["final_fp"] = fullrun.fingerprints(Q, r)
        fix["final_linf"] = float(np.abs(Q).max())
    np.savez_compressed(os.path.join(out, f"full_{name}.npz"), **fix)
    if name == "cfg3":
        np.savez_compressed(os.path.join(out, "refarm_cfg3.npz"), q=np.array(strata_q),
                            step=np.array(strata_step), iterations=np.array(strata_its), dt=np.array(rec["dt"]),
                            hist=np.array(rec["hist"]))
    return {"config": name, "steps": len(rec["dt"]), "wall_s": time.time() - t0,
            "first_nonfinite_step": first_nonfinite}


def fv_volumes(P):
    """(volumes, m) view of FV patches (B, m, k, k, k): one row per finite volume."""
    B, m = P.shape[:2]
    return P.transpose(0, 2, 3, 4, 1).reshape(-1, m)


def fv_run(procs, out):
    cfg = cf.CONFIGS["cfg4"]
    t0 = time.time()
    P = cf.initial_fv(cfg)
    dts = []
    with fullrun.pool_for(cfg, procs) as pool:
        for k in range(cfg.steps):
            P, dt = fullrun.fv_step(pool, cfg, P, 4 * procs)
            dts.append(dt)
            if k % 10 == 9:
                print(f"cfg4 step {k + 1}/{cfg.steps} t={time.time() - t0:.0f}s", flush=True)
    dts = np.array(dts)
    vols = fv_volumes(P)
    sample = sample_cells(vols.shape[0])
    np.savez_compressed(os.path.join(out, "full_cfg4.npz"), config="cfg4", steps_run=cfg.steps, dt=dts,
                        sha256_state=hashlib.sha256(np.ascontiguousarray(P).tobytes()).hexdigest(),
                        sha256_dt=hashlib.sha256(dts.tobytes()).hexdigest(), sample=sample,
                        final_sample=vols[sample], integrals=P.sum(axis=(0, 2, 3, 4)) / cfg.cells ** 3)
    return {"config": "cfg4", "steps": cfg.steps, "wall_s": time.time() - t0}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="cfg2s,cfg2,cfg5,cfg4,cfg3")
    ap.add_argument("--procs", type=int, default=os.cpu_count() or 4)
    ap.add_argument("--out", default=HERE)
    a = ap.parse_args()
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    for name in a.configs.split(","):
        res = fv_run(a.procs, a.out) if name == "cfg4" else dg_run(name, a.procs, a.out)
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
