"""Cell-batched restatement of the per-cell oracle (oracle only).

Same arithmetic as `oracle.ops` (and hence reference kernels.py) with a
leading cell axis C: Q has shape (C, m, n, ..., n).  The space-time iterate is
kept as (n_t, C, m, ...), i.e. the per-cell (n_t, m, ...) with C inserted after
the time axis, so every tensordot contracts the same-length axis as the
per-cell code.  A per-cell active mask reproduces the reference's per-cell
early exit (kernels.py:139-147).  tests/test_oracle_golden.py checks this
module bit-for-bit against `oracle.ops` on cell subsets.
"""
from __future__ import annotations

import numpy as np

from .ops import time_operators, rusanov


def _flux_b(pde, Q, a):
    """Pointwise flux of a (C, m, ...) batch: the plugin wants (m, ...)."""
    return np.moveaxis(pde.flux(np.moveaxis(Q, 1, 0), a), 0, 1)


def _lam_b(pde, Q, a):
    return pde.max_eigenvalue(np.moveaxis(Q, 1, 0), a)


def nodal_divergence_b(Q, pde, basis, edges):
    """kernels.py:63-70 with a cell axis (contraction axis shifted by one)."""
    acc = np.zeros_like(Q)
    for a in range(Q.ndim - 2):
        fa = _flux_b(pde, Q, a)
        acc += np.moveaxis(np.tensordot(basis.diff_matrix, fa, axes=(1, 2 + a)), 0, 2 + a) / edges[a]
    return acc


def face_traces_b(V, basis):
    """kernels.py:73-79 batched: {(a, s): (C, m, n^(d-1))}."""
    d = V.ndim - 2
    return {(a, s): np.tensordot(basis.trace(s), V, axes=(0, 2 + a))
            for a in range(d) for s in (0, 1)}


def predictor_picard_b(Q, pde, dt, basis, edges, tol=1e-10, max_iter=None):
    """kernels.py:120-159 over a batch.  Returns dict of arrays:
    q_int, q_end (C, m, ...), trace_q / trace_f {(a,s): (C, m, ...)},
    iterations (C,) int, converged (C,) bool.

    `dt` may be a scalar or a per-cell array (C,) -- the latter only for the
    reference-arm sampler; the Algorithm-1 drivers always pass a scalar.
    """
    if max_iter is None:
        max_iter = 2 * basis.n
    kinv, lift = time_operators(basis)
    nt = basis.n
    w = basis.weights
    C = Q.shape[0]
    qhat = np.repeat(Q[None], nt, axis=0)
    base = np.tensordot(kinv @ lift[:, None], Q[None], axes=(1, 0))
    its = np.zeros(C, dtype=np.int64)
    done = np.zeros(C, dtype=bool)
    active = np.arange(C)
    for it in range(1, max_iter + 1):
        its[active] = it
        qa = qhat[:, active]
        rhs = np.stack([-dt * w[r] * nodal_divergence_b(qa[r], pde, basis, edges) for r in range(nt)])
        nxt = base[:, active] + np.tensordot(kinv, rhs, axes=(1, 0))
        delta = np.abs(nxt - qa).reshape(nt, len(active), -1).max(axis=(0, 2))
        qhat[:, active] = nxt
        ok = delta < tol
        done[active[ok]] = True
        active = active[~ok]
        if active.size == 0:
            break
    return _epilogue_b(Q.ndim - 2, qhat, pde, dt, basis, its, done)


def _epilogue_b(d, qhat, pde, dt, basis, its, done):
    """kernels.py:148-159 batched."""
    w = basis.weights
    q_end = np.tensordot(basis.trace_right, qhat, axes=(0, 0))
    q_int = dt * np.tensordot(w, qhat, axes=(0, 0))
    tq = face_traces_b(q_int, basis)
    tf = {}
    for a in range(d):
        fn = np.stack([_flux_b(pde, qhat[r], a) for r in range(basis.n)])
        fi = dt * np.tensordot(w, fn, axes=(0, 0))
        for s in (0, 1):
            tf[(a, s)] = np.tensordot(basis.trace(s), fi, axes=(0, 2 + a))
    return dict(q_int=q_int, q_end=q_end, trace_q=tq, trace_f=tf,
                iterations=its, converged=done)


def rusanov_b(lo, hi, pde, axis, sign=1):
    """kernels.py:162-173 on (F, m, ...) face batches."""
    return np.moveaxis(rusanov(np.moveaxis(lo, 1, 0), np.moveaxis(hi, 1, 0), pde, axis, sign), 0, 1)


def correct_b(q_end, trace_f, outcomes, basis, edges):
    """kernels.py:176-193 batched; outcomes/trace_f: {(a,s): (C, m, ...)}."""
    q = q_end.copy()
    for a in range(q.ndim - 2):
        for s in (0, 1):
            jump = outcomes[(a, s)] - trace_f[(a, s)]
            sgn = 1.0 if s == 1 else -1.0
            lift = sgn * basis.trace(s) / (basis.weights * edges[a])
            # per cell: moveaxis(tensordot(lift, jump_c, axes=0), 0, 1 + a)
            q -= np.moveaxis(np.tensordot(lift, jump, axes=0), 0, 2 + a)
    return q


def cell_speed_b(Q, pde, dim):
    """Per-cell lambda of kernels.py:271-273 for a batch: numpy max over nodes
    propagates NaN per axis; the Python max over axes drops a NaN axis."""
    C = Q.shape[0]
    lam = np.zeros(C)
    for a in range(dim):
        ax = _lam_b(pde, Q, a).reshape(C, -1).max(axis=1)
        take = ax > lam            # Python max(lam, ax): ax only if strictly greater
        lam = np.where(take, ax, lam)
    return lam


def stable_dt_b(Q, h, pde, order, cfl, dim):
    """kernels.py:267-281 for a batch with per-cell h (C,) or scalar h."""
    lam = cell_speed_b(Q, pde, dim)
    hh = np.broadcast_to(np.asarray(h, dtype=float), lam.shape)
    keep = lam > 0.0
    if not keep.any():
        from .ops import OracleNoWaveSpeed
        raise OracleNoWaveSpeed("no positive wave speed anywhere; cannot pick a time step")
    cand = hh[keep] / ((2 * order + 1) * lam[keep])
    return cfl * float(cand.min())


def fv_update_b(P, pde, dt, edges, halos):
    """kernels.py:225-253 over a batch of patches (B, m, k, ...);
    halos {(a,s): (B, m, k^(d-1))}."""
    d = P.ndim - 2
    k = P.shape[2]
    out = P.copy()
    for a in range(d):
        dx = edges[a] / k
        ext = np.concatenate([np.expand_dims(halos[(a, 0)], 2 + a), P,
                              np.expand_dims(halos[(a, 1)], 2 + a)], axis=2 + a)
        ext = np.moveaxis(ext, 2 + a, 2)
        fl = [rusanov_b(ext[:, :, i], ext[:, :, i + 1], pde, a) for i in range(k + 1)]
        view = np.moveaxis(out, 2 + a, 2)
        for i in range(k):
            view[:, :, i] -= (dt / dx) * (fl[i + 1] - fl[i])
    return out
