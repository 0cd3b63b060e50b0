"""Full-size Algorithm-1 runs of the batched oracle over a process pool
(oracle only: test infrastructure for tests/golden/make_full_parity.py and
tools/parity_report.py).

The predictor (kernels.py:120-159, restated cell-batched in
oracle/batched.py) is farmed out to worker processes in contiguous cell
chunks; the face solves (kernels.py:162-173), the corrector
(kernels.py:176-193) and the dt reduction (kernels.py:267-281) run in the
parent.  Splitting the batch changes nothing numerically: every batched
kernel is cell-independent.
"""
from __future__ import annotations

import os

import numpy as np

from . import batched, drivers, ops

_W = {}


def make_pde(name, dim, velocity=(1.0, 0.5)):
    return ops.advection(velocity, dim) if name == "advection" else ops.make_pde(name, dim=dim)


def init_worker(name, dim, velocity, order):
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    _W["pde"] = make_pde(name, dim, velocity)
    _W["basis"] = ops.basis_for(order)


def _stp_chunk(args):
    Q, dt, edges = args
    return batched.predictor_picard_b(Q, _W["pde"], dt, _W["basis"], edges)


def _stp_cell(args):
    q, dt, edges = args
    return ops.predictor_picard(q, _W["pde"], dt, _W["basis"], edges)


def _fv_chunk(args):
    P, dt, edges, halos = args
    return batched.fv_update_b(P, _W["pde"], dt, edges, halos)


def pool_for(cfg, procs):
    import multiprocessing as mp
    ctx = mp.get_context("fork")
    return ctx.Pool(procs, initializer=init_worker, initargs=(cfg.pde, cfg.dim, cfg.velocity, max(cfg.order, 1)))


def uniform_step(pool, cfg, Q, nchunks):
    """One Algorithm-1 step on the uniform grid; returns (Q_next, dt, iterations)."""
    pde = make_pde(cfg.pde, cfg.dim, cfg.velocity)
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


def fv_step(pool, cfg, P, nchunks):
    pde = make_pde("euler", 3)
    h = 1.0 / cfg.cells
    edges = (h * cfg.patch,) * 3
    dt = drivers.fv_dt(P, pde, cfg.cfl, h)
    halos = drivers.fv_halos(P)
    idx = np.array_split(np.arange(P.shape[0]), nchunks)
    parts = pool.map(_fv_chunk, [(P[i], dt, edges, {k: v[i] for k, v in halos.items()}) for i in idx])
    return np.concatenate(parts), dt


def amr_step(pool, cfg, forest, Q, sweep):
    """One Algorithm-1 step on the static adaptive mesh (per-cell kernels,
    oracle/drivers.py dg_amr_step with the predictor in the pool).
    Q: (C, m, n^d) in forest.sfc order."""
    from . import transfer
    pde = make_pde(cfg.pde, cfg.dim, cfg.velocity)
    basis = ops.basis_for(cfg.order)
    ops_t = transfer.transfer_for(cfg.order)
    d = cfg.dim
    keys = forest.sfc
    dt = ops.stable_dt(((min(forest.cell_edges(k[0])), Q[i]) for i, k in enumerate(keys)), pde, cfg.order,
                       cfg.cfl, d)
    stl = pool.map(_stp_cell, [(Q[i], dt, forest.cell_edges(k[0])) for i, k in enumerate(keys)], chunksize=256)
    stores = dict(zip(keys, stl))
    outcome = drivers.amr_face_outcomes(forest, stores, pde, ops_t, sweep)
    Qn = np.stack([ops.correct(stores[k], {(a, sd): outcome[forest.side_face_key(k, a, sd)]
                                            for a in range(d) for sd in (0, 1)}, basis, forest.cell_edges(k[0]))
                   for k in keys])
    its = np.array([stores[k].iterations for k in keys])
    return Qn, dt, its


# ------------------------------------------------------------ fixtures ---

def fingerprint_weights(seed, shape):
    """Per-cell fingerprint weights r in [0.5, 1.5) over one cell's (m, n^d)
    block: f_c = sum(r * Q_c).  A deviation in any single DoF of any cell moves
    that cell's fingerprint (all weights are positive and distinct)."""
    return np.random.default_rng(seed).uniform(0.5, 1.5, size=shape)


def fingerprints(Q, r):
    C = Q.shape[0]
    return Q.reshape(C, -1) @ r.reshape(-1)


def integrals(Q, weights_nd, volume):
    """Conserved integrals per component: sum_c vol_c * sum_nodes w * Q_c."""
    C, m = Q.shape[:2]
    vol = np.broadcast_to(np.asarray(volume, dtype=float), (C,))
    per = (Q.reshape(C, m, -1) * weights_nd.reshape(1, 1, -1)).sum(axis=2)
    return (per * vol[:, None]).sum(axis=0)


def tensor_weights(w, dim):
    out = w
    for _ in range(dim - 1):
        out = np.multiply.outer(out, w)
    return out
