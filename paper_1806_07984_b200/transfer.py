"""3:1 face transfer on the GPU -- mirror of
/root/reference/pkg/src/enclavedg/transfer.py:18-96.

TransferOperators / get_transfer keep the reference attributes (interp,
restrict lists of n x n numpy matrices, built exactly like transfer.py:28-39);
the functions run the sm_100a face-transfer kernel of libenclavedg_b200.
"""
from __future__ import annotations

import ctypes as C
import threading

import numpy as np

from . import _lib
from .basis import get_basis
from .errors import NotReadyError
from .kernels import _dev, _stream, _torch


class TransferOperators:
    """interp[j] / restrict[j] between a parent interval and its thirds."""

    def __init__(self, order: int):
        self.order = order
        self.basis = get_basis(order)
        interp, restr = self.basis.transfer_matrices()
        self.interp = list(interp)
        self.restrict = list(restr)


_OPS_CACHE: dict = {}


def get_transfer(order: int) -> TransferOperators:
    if order not in _OPS_CACHE:
        _OPS_CACHE[order] = TransferOperators(order)
    return _OPS_CACHE[order]


def _apply(ops: TransferOperators, data, child_pos, restrict_mode: int):
    torch = _torch()
    x, host = _dev(data)
    dim = x.dim()                 # trace (m, n^(d-1)) of a d-D cell
    if len(child_pos) != dim - 1:
        raise ValueError("child_pos needs one digit per transverse axis")
    m = x.shape[0]
    cp = torch.tensor([list(child_pos) + [0] * (2 - len(child_pos))], dtype=torch.int8, device="cuda")
    out = torch.empty_like(x)
    _lib.check(_lib.load().edg_interpolate_face_trace(dim, m, ops.order, _lib.ptr(ops.basis.device_table()), 1,
                                                      _lib.ptr(x), _lib.ptr(cp), restrict_mode, _lib.ptr(out),
                                                      _stream()), "face transfer")
    return out.cpu().numpy() if host else out


def interpolate_face_trace(ops: TransferOperators, trace, child_pos):
    """transfer.py:59-66."""
    return _apply(ops, trace, tuple(child_pos), 0)


def restrict_face_values(ops: TransferOperators, values, child_pos):
    """transfer.py:69-72."""
    return _apply(ops, values, tuple(child_pos), 1)


def interpolate_to_virtual(ops: TransferOperators, parent_trace, child_pos, stp_complete=True):
    """transfer.py:75-79 -- the parent predictor must be complete."""
    if not stp_complete:
        raise NotReadyError("parent predictor incomplete; trace interpolation must wait")
    return interpolate_face_trace(ops, parent_trace, child_pos)


def restrict_riemann(ops: TransferOperators, buffers, child_outcome, child_pos, sweep):
    """transfer.py:82-96: zero-init per sweep, refuse a double restriction,
    accumulate restrict[child_pos] (x) child_outcome into buffers.outcome."""
    guard = getattr(buffers, "write_guard", None) or threading.Lock()
    with guard:
        if buffers.accum_sweep != sweep:
            buffers.accum_sweep = sweep
            buffers.outcome = np.zeros_like(np.asarray(child_outcome)) if isinstance(child_outcome, np.ndarray) \
                else _torch().zeros_like(child_outcome)
            buffers.restricted_children = set()
        if child_pos in buffers.restricted_children:
            raise AssertionError(f"child {child_pos} restricted twice in sweep {sweep}")
        buffers.restricted_children.add(child_pos)
        buffers.outcome += restrict_face_values(ops, child_outcome, child_pos)


def face_transfer_batch(order: int, traces, child_pos, restrict_mode: bool):
    """Batched interpolate/restrict: traces (F, m, n^(d-1)), child_pos (F, 2) int8."""
    torch = _torch()
    x, _ = _dev(traces)
    F_, m = x.shape[:2]
    dim = x.dim() - 1
    out = torch.empty_like(x)
    b = get_basis(order)
    _lib.check(_lib.load().edg_interpolate_face_trace(dim, m, order, _lib.ptr(b.device_table()), F_, _lib.ptr(x),
                                                      _lib.ptr(child_pos), int(restrict_mode), _lib.ptr(out),
                                                      _stream()), "face transfer")
    return out


# --------------------------------------------------------------------------
# Cell-local operators of dynamic AMR:
# transfer.py:99-158 of the reference on the sm_100a kernels of
# csrc/edg_amr.cuh.  The mesh mutation (plan_mesh_updates /
# apply_mesh_updates, transfer.py:161-219) is host-side topology work and
# lives in amr.py, which calls these operators to migrate the state.

def _vol_dev(x):
    x, host = _dev(x)
    if x.dim() not in (3, 4):
        raise ValueError("cell data must be (m, n, n[, n])")
    return x, host


def interpolate_volume_batch(order: int, Q, digits, parent=None):
    """Children of parents: out[i] = interpolate_volume(Q[parent[i]], digits[i]).
    Q (C, m, n^d...) on the GPU, digits (I, dim) ints in {0, 1, 2}, parent (I,)
    or None (item i uses cell i)."""
    torch = _torch()
    x, _ = _dev(Q)
    dim = x.dim() - 2
    C_, m = x.shape[:2]
    dg = torch.as_tensor(np.asarray(digits), dtype=torch.int8).reshape(-1, dim)
    if dg.numel() and (int(dg.min()) < 0 or int(dg.max()) > 2):
        raise ValueError("child digits must be 0, 1 or 2")
    ni = dg.shape[0]
    d3 = torch.zeros((ni, 3), dtype=torch.int8)
    d3[:, :dim] = dg
    d3 = d3.cuda()
    par = None
    if parent is not None:
        par = torch.as_tensor(np.asarray(parent), dtype=torch.int32).reshape(-1).cuda()
        if par.numel() != ni:
            raise ValueError("one parent index per item")
    elif ni != C_:
        raise ValueError("without parent indices, one item per cell")
    out = torch.empty((ni,) + tuple(x.shape[1:]), dtype=torch.float64, device="cuda")
    b = get_basis(order)
    _lib.check(_lib.load().edg_interpolate_volume(dim, m, order, _lib.ptr(b.device_table()), ni,
                                                  None if par is None else _lib.ptr(par), _lib.ptr(x),
                                                  _lib.ptr(d3), _lib.ptr(out), _stream()), "interpolate_volume")
    return out


def interpolate_volume(ops: TransferOperators, q, child_digits):
    """transfer.py:99-102: the cell polynomial on one volumetric child."""
    x, host = _vol_dev(q)
    out = interpolate_volume_batch(ops.order, x[None], [tuple(child_digits)])[0]
    return out.cpu().numpy() if host else out


def restrict_volume_batch(order: int, children):
    """children (P, 3^d, m, n^d...) in row-major digit order -> (P, m, n^d...)."""
    torch = _torch()
    x, _ = _dev(children)
    dim = x.dim() - 3
    P_, nch, m = x.shape[:3]
    if nch != 3 ** dim:
        raise ValueError("need all 3^d children per parent")
    out = torch.empty((P_,) + tuple(x.shape[2:]), dtype=torch.float64, device="cuda")
    b = get_basis(order)
    _lib.check(_lib.load().edg_restrict_volume(dim, m, order, _lib.ptr(b.device_table()), P_, _lib.ptr(x),
                                               _lib.ptr(out), _stream()), "restrict_volume")
    return out


def restrict_volume(ops: TransferOperators, children: dict):
    """transfer.py:105-118: L2 projection of the 3^d children onto the parent.
    The children are summed in the dict's order, like the reference."""
    torch = _torch()
    keys = list(children.keys())
    dim = len(keys[0])
    if len(keys) != 3 ** dim:
        raise ValueError("need all 3^d children")
    first, host = _vol_dev(children[keys[0]])
    # the kernel sums in row-major digit order; other dict orders are
    # summed here child by child in the caller's order
    order_rm = list(np.ndindex(*(3,) * dim))
    if keys == order_rm:
        stack = torch.stack([_dev(children[k])[0] for k in keys])[None]
        out = restrict_volume_batch(ops.order, stack)[0]
    else:
        out = None
        for k in keys:
            part = _restrict_one(ops, _dev(children[k])[0], k)
            out = part if out is None else out + part
    return out.cpu().numpy() if host else out


def _restrict_one(ops, q, digits):
    """restrict[digits] contraction of one child: the interpolation kernel
    with the restriction matrices (the parent is the only 'child')."""
    torch = _torch()
    dim = len(digits)
    z = torch.zeros((3 ** dim,) + tuple(q.shape), dtype=torch.float64, device="cuda")
    z[int(np.ravel_multi_index(digits, (3,) * dim))] = q
    return restrict_volume_batch(ops.order, z[None])[0]


def gradient_indicator_batch(Q, order: int, levels=None, decision=None, min_level: int = 0):
    """transfer.py:136-158 on a batch (C, m, n^d...): indicator per cell, and
    with a RefinementDecision the verdicts (+1 refine, 0 keep, -1 coarsen)."""
    torch = _torch()
    x, _ = _dev(Q)
    dim = x.dim() - 2
    C_, m = x.shape[:2]
    ind = torch.empty(C_, dtype=torch.float64, device="cuda")
    verdict = lv = None
    rt, ct, ml = 0.0, 0.0, 0
    if decision is not None:
        verdict = torch.empty(C_, dtype=torch.int8, device="cuda")
        rt, ct, ml = float(decision.refine_tol), float(decision.coarsen_tol), int(decision.max_level)
        if levels is not None:
            lv = torch.as_tensor(np.asarray(levels), dtype=torch.int32).reshape(-1).cuda()
    b = get_basis(order)
    _lib.check(_lib.load().edg_gradient_indicator(dim, m, order, _lib.ptr(b.device_table()), C_, _lib.ptr(x),
                                                  None if lv is None else _lib.ptr(lv), rt, ct, ml, int(min_level),
                                                  _lib.ptr(ind), None if verdict is None else _lib.ptr(verdict),
                                                  _stream()), "gradient_indicator")
    return ind if verdict is None else (ind, verdict)


def gradient_indicator(q, order: int) -> float:
    """transfer.py:136-148: max |reference-space derivative| of one cell."""
    x, _ = _vol_dev(q)
    return float(gradient_indicator_batch(x[None], order)[0].item())


class RefinementDecision:
    """Hysteresis band of the refinement criterion (transfer.py:121-133):
    verdict strings REFINE / KEEP / COARSEN; refine_tol > coarsen_tol >= 0."""
    REFINE = "refine"
    KEEP = "keep"
    COARSEN = "coarsen"

    def __init__(self, refine_tol: float, coarsen_tol: float, max_level: int):
        if not refine_tol > coarsen_tol >= 0:
            raise ValueError("need refine_tol > coarsen_tol >= 0 (hysteresis band)")
        self.refine_tol, self.coarsen_tol, self.max_level = refine_tol, coarsen_tol, max_level


_VERDICT = {1: RefinementDecision.REFINE, 0: RefinementDecision.KEEP, -1: RefinementDecision.COARSEN}


def evaluate_refinement_criterion(q, level, order, decision: RefinementDecision, min_level):
    """transfer.py:151-158: the verdict from the cell's own coefficients."""
    x, _ = _vol_dev(q)
    _, v = gradient_indicator_batch(x[None], order, [level], decision, min_level)
    return _VERDICT[int(v[0].item())]
