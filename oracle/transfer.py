"""3:1 inter-resolution transfer restatement (oracle only).

Follows /root/reference/pkg/src/enclavedg/transfer.py:18-118.
"""
from __future__ import annotations

import numpy as np

from .ops import basis_for, OracleNotReady


class Transfer:
    """interp[j]: parent polynomial at child-j GL points; restrict[j]: its
    GL-inner-product adjoint with child measure 1/3 (transfer.py:18-39)."""

    def __init__(self, order: int):
        b = basis_for(order)
        self.order = order
        self.basis = b
        w = b.weights
        self.interp, self.restrict = [], []
        for j in range(3):
            e = b.lagrange_eval((j + b.nodes) / 3.0)
            self.interp.append(e)
            self.restrict.append((e.T * w[None, :]) / w[:, None] / 3.0)


_CACHE: dict = {}


def transfer_for(order: int) -> Transfer:
    if order not in _CACHE:
        _CACHE[order] = Transfer(order)
    return _CACHE[order]


def along_axes(mats, data, axes):
    """Contract one square matrix per listed array axis (transfer.py:51-56)."""
    out = data
    for mat, ax in zip(mats, axes):
        out = np.moveaxis(np.tensordot(mat, out, axes=(1, ax)), 0, ax)
    return out


def interp_trace(ops: Transfer, trace, child_pos):
    """transfer.py:59-66."""
    return along_axes([ops.interp[j] for j in child_pos], trace, range(1, 1 + len(child_pos)))


def restrict_trace(ops: Transfer, values, child_pos):
    """transfer.py:69-72."""
    return along_axes([ops.restrict[j] for j in child_pos], values, range(1, 1 + len(child_pos)))


def to_virtual(ops: Transfer, parent_trace, child_pos, stp_complete=True):
    """transfer.py:75-79."""
    if not stp_complete:
        raise OracleNotReady("parent predictor incomplete; trace interpolation must wait")
    return interp_trace(ops, np.asarray(parent_trace, dtype=float), child_pos)


class ParentAccumulator:
    """The caller-owned `buffers` object restrict_riemann expects
    (transfer.py:88-96): sweep tag, running outcome, children seen."""

    def __init__(self):
        self.accum_sweep = None
        self.outcome = None
        self.restricted_children = set()


def accumulate_restriction(ops: Transfer, buf: ParentAccumulator, child_outcome, child_pos, sweep):
    """transfer.py:82-96 (no lock needed: the oracle is single threaded)."""
    if buf.accum_sweep != sweep:
        buf.accum_sweep = sweep
        buf.outcome = np.zeros_like(child_outcome)
        buf.restricted_children = set()
    if child_pos in buf.restricted_children:
        raise AssertionError(f"child {child_pos} restricted twice in sweep {sweep}")
    buf.restricted_children.add(child_pos)
    buf.outcome += restrict_trace(ops, child_outcome, child_pos)


def interp_volume(ops: Transfer, q, digits):
    """transfer.py:99-102."""
    return along_axes([ops.interp[j] for j in digits], q, range(1, 1 + len(digits)))


def restrict_volume(ops: Transfer, children: dict):
    """transfer.py:105-118."""
    out = None
    d = len(next(iter(children.keys())))
    for digits, q in children.items():
        part = along_axes([ops.restrict[j] for j in digits], q, range(1, 1 + d))
        out = part if out is None else out + part
    return out


def gradient_indicator(q, order: int) -> float:
    """transfer.py:136-148: the largest |reference-space derivative| over the
    nodes, components and axes (np.max per axis propagates NaN, the Python
    max over axes drops a NaN axis)."""
    D = basis_for(order).diff_matrix
    worst = 0.0
    for ax in range(q.ndim - 1):
        g = np.moveaxis(np.tensordot(D, q, axes=(1, 1 + ax)), 0, 1 + ax)
        worst = max(worst, float(np.abs(g).max()))
    return worst


REFINE, KEEP, COARSEN = 1, 0, -1


def refinement_verdict(q, level, order, refine_tol, coarsen_tol, max_level, min_level) -> int:
    """transfer.py:151-158 as +1 refine / 0 keep / -1 coarsen."""
    ind = gradient_indicator(q, order)
    if ind > refine_tol and level < max_level:
        return REFINE
    if ind < coarsen_tol and level > min_level:
        return COARSEN
    return KEEP
