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
