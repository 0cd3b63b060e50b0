"""Reference-API mirror of the cell/face kernels, executed on the B200.

Same names, signatures, return types and error behaviour as
/root/reference/pkg/src/enclavedg/kernels.py: stp_picard (:120), project_to_faces
(:73), riemann_rusanov (:162), corrector (:176), fv_patch_update (:225),
patch_boundary_layers (:256), admissible_dt (:267), PredictorStore (:25),
CellSolution (:44).  Inputs may be numpy arrays (results come back as numpy,
so the functions drop into reference call sites) or float64 CUDA tensors
(results stay on the device).  Every computation runs in the sm_100a kernels
of libenclavedg_b200 through the C ABI; there is no CPU path.

The *_batch variants are the native form: a leading cell (or face / patch)
axis, device tensors in and out, asynchronous on the current stream.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .basis import PolynomialBasis, get_basis
from .errors import ConfigError, EnclaveDgError, NativeError, NotReadyError
from .pde import PdeDescriptor


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise NativeError("no CUDA device visible: the enclavedg_b200 kernels have no CPU fallback")
    return torch


def _stream():
    torch = _torch()
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _dev(x):
    """(float64 contiguous CUDA tensor, came_from_numpy)."""
    torch = _torch()
    if isinstance(x, torch.Tensor):
        t = x.to(device="cuda", dtype=torch.float64)
        return t.contiguous(), False
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).cuda(), True


def _scalar_dev(v):
    torch = _torch()
    if isinstance(v, torch.Tensor):
        return v.to(device="cuda", dtype=torch.float64).reshape(1).contiguous()
    return torch.tensor([float(v)], dtype=torch.float64, device="cuda")


def _edges_dev(edges, dim, ncells):
    """(device tensor, per_cell flag) for a tuple or a (C, dim) array."""
    torch = _torch()
    if isinstance(edges, torch.Tensor) and edges.dim() == 2:
        return edges.to(device="cuda", dtype=torch.float64).contiguous(), 1
    e = np.asarray(edges, dtype=np.float64)
    if e.ndim == 2:
        return torch.from_numpy(np.ascontiguousarray(e)).cuda(), 1
    if e.shape != (dim,):
        raise ConfigError(f"edges must have {dim} entries")
    return torch.from_numpy(e.copy()).cuda(), 0


def trace_keys(dim):
    return [(a, s) for a in range(dim) for s in (0, 1)]


@dataclass
class PredictorStore:
    """Per-cell predictor results (kernels.py:25-41)."""

    q_int: object
    q_end: object
    trace_q: dict
    trace_f: dict
    iterations: int = 0
    converged: bool = True
    checksum: float | None = None


class CellSolution:
    """DG coefficients plus the completion marker (kernels.py:44-60).  On the
    GPU the marker is a CUDA event / stream order."""

    __slots__ = ("key", "q", "stp_complete", "klass", "predictor", "task_state")

    def __init__(self, key, q):
        self.key = key
        self.q = q
        self.stp_complete = True
        self.klass = "enclave"
        self.predictor = None
        self.task_state = "idle"


def _check_supported(pde: PdeDescriptor, order: int):
    if not _lib.load().edg_supported(C.byref(pde.native()), order):
        raise ConfigError(f"order {order} of {pde.name} in {pde.dim}-D is not built into libenclavedg_b200")


# ------------------------------------------------------------- predictor --

def stp_picard_batch(Q, pde: PdeDescriptor, dt, basis: PolynomialBasis, edges, tol=1e-10, max_iter=None,
                     cell_list=None, out=None, want_q_int=True):
    """Picard STP of many cells (kernels.py:120-159 per cell).

    Q: (C, m, n^d) float64 CUDA tensor; dt: float or device scalar; edges:
    tuple (shared) or (C, dim).  cell_list: optional int32 device tensor of
    the cells to process.  Returns dict q_int, q_end (C, m, n^d), trace_q,
    trace_f (C, 2d, m, n^(d-1)), iterations (C,) int32, converged (C,) uint8.
    """
    torch = _torch()
    lib = _lib.load()
    _check_supported(pde, basis.order)
    Qd, _ = _dev(Q)
    C_ = Qd.shape[0]
    d, m, n = pde.dim, pde.m, basis.n
    if Qd.shape[1:] != (m,) + (n,) * d:
        raise ConfigError(f"q must be (C, {m}) + ({n},)*{d}, got {tuple(Qd.shape)}")
    if out is None:
        out = dict(
            q_end=torch.empty_like(Qd),
            q_int=torch.empty_like(Qd) if want_q_int else None,
            trace_q=torch.empty((C_, 2 * d, m) + (n,) * (d - 1), dtype=torch.float64, device="cuda"),
            trace_f=torch.empty((C_, 2 * d, m) + (n,) * (d - 1), dtype=torch.float64, device="cuda"),
            iterations=torch.zeros(C_, dtype=torch.int32, device="cuda"),
            converged=torch.zeros(C_, dtype=torch.uint8, device="cuda"))
    e, per = _edges_dev(edges, d, C_)
    dtd = _scalar_dev(dt)
    nwork = C_ if cell_list is None else int(cell_list.numel())
    st = lib.edg_stp_picard(C.byref(pde.native()), basis.order, _lib.ptr(basis.device_table()), _lib.ptr(Qd),
                            _lib.ptr(cell_list), nwork, _lib.ptr(e), per, _lib.ptr(dtd), float(tol),
                            0 if max_iter is None else int(max_iter), _lib.ptr(out["q_end"]),
                            _lib.ptr(out["q_int"]), _lib.ptr(out["trace_q"]), _lib.ptr(out["trace_f"]),
                            _lib.ptr(out["iterations"]), _lib.ptr(out["converged"]), None, _stream())
    _lib.check(st, "stp_picard")
    return out


def stp_picard(q, pde: PdeDescriptor, dt, basis: PolynomialBasis, edges, tol=1e-10, max_iter=None) -> PredictorStore:
    """Drop-in for kernels.py:120-159 on one cell."""
    Qd, host = _dev(q)
    r = stp_picard_batch(Qd[None], pde, dt, basis, tuple(edges), tol, max_iter)
    conv = lambda t: t.cpu().numpy() if host else t  # noqa: E731
    keys = trace_keys(pde.dim)
    return PredictorStore(conv(r["q_int"][0]), conv(r["q_end"][0]),
                          {k: conv(r["trace_q"][0, j]) for j, k in enumerate(keys)},
                          {k: conv(r["trace_f"][0, j]) for j, k in enumerate(keys)},
                          iterations=int(r["iterations"][0]), converged=bool(r["converged"][0]))


def stp_linear_batch(Q, pde: PdeDescriptor, dt, basis: PolynomialBasis, edges, cell_list=None):
    """Cauchy-Kowalevski predictor of many cells (kernels.py:82-106 per cell);
    same outputs as stp_picard_batch (iterations 0, converged 1)."""
    torch = _torch()
    if not pde.is_linear:
        raise EnclaveDgError("stp_linear requires a linear flux")
    _check_supported(pde, basis.order)
    Qd, _ = _dev(Q)
    C_ = Qd.shape[0]
    d, m, n = pde.dim, pde.m, basis.n
    out = dict(q_end=torch.empty_like(Qd), q_int=torch.empty_like(Qd),
               trace_q=torch.empty((C_, 2 * d, m) + (n,) * (d - 1), dtype=torch.float64, device="cuda"),
               trace_f=torch.empty((C_, 2 * d, m) + (n,) * (d - 1), dtype=torch.float64, device="cuda"),
               iterations=torch.zeros(C_, dtype=torch.int32, device="cuda"),
               converged=torch.zeros(C_, dtype=torch.uint8, device="cuda"))
    e, per = _edges_dev(edges, d, C_)
    dtd = _scalar_dev(dt)
    nwork = C_ if cell_list is None else int(cell_list.numel())
    st = _lib.load().edg_stp_linear(C.byref(pde.native()), basis.order, _lib.ptr(basis.device_table()),
                                    _lib.ptr(Qd), _lib.ptr(cell_list), nwork, _lib.ptr(e), per, _lib.ptr(dtd),
                                    _lib.ptr(out["q_end"]), _lib.ptr(out["q_int"]), _lib.ptr(out["trace_q"]),
                                    _lib.ptr(out["trace_f"]), _lib.ptr(out["iterations"]), _lib.ptr(out["converged"]),
                                    _stream())
    _lib.check(st, "stp_linear")
    return out


def stp_linear(q, pde: PdeDescriptor, dt, basis: PolynomialBasis, edges) -> PredictorStore:
    """Drop-in for kernels.py:82-106 on one cell."""
    Qd, host = _dev(q)
    r = stp_linear_batch(Qd[None], pde, dt, basis, tuple(edges))
    conv = lambda t: t.cpu().numpy() if host else t  # noqa: E731
    keys = trace_keys(pde.dim)
    return PredictorStore(conv(r["q_int"][0]), conv(r["q_end"][0]),
                          {k: conv(r["trace_q"][0, j]) for j, k in enumerate(keys)},
                          {k: conv(r["trace_f"][0, j]) for j, k in enumerate(keys)})


def project_to_faces_batch(V, basis: PolynomialBasis, dim: int):
    torch = _torch()
    Vd, _ = _dev(V)
    C_, m = Vd.shape[:2]
    n = basis.n
    out = torch.empty((C_, 2 * dim, m) + (n,) * (dim - 1), dtype=torch.float64, device="cuda")
    _lib.check(_lib.load().edg_project_to_faces(dim, m, basis.order, _lib.ptr(basis.device_table()), C_,
                                                _lib.ptr(Vd), _lib.ptr(out), _stream()), "project_to_faces")
    return out


def project_to_faces(q_vol, basis: PolynomialBasis):
    """Drop-in for kernels.py:73-79."""
    Vd, host = _dev(q_vol)
    dim = Vd.dim() - 1
    r = project_to_faces_batch(Vd[None], basis, dim)[0]
    return {k: (r[j].cpu().numpy() if host else r[j]) for j, k in enumerate(trace_keys(dim))}


# --------------------------------------------------------------- Riemann --

def riemann_rusanov(trace_lo, trace_hi, pde: PdeDescriptor, axis, sign=1):
    """Drop-in for kernels.py:162-173 (pointwise; any trailing shape)."""
    torch = _torch()
    lo, host = _dev(trace_lo)
    hi, _ = _dev(trace_hi)
    if lo.shape != hi.shape or lo.shape[0] != pde.m:
        raise ConfigError("trace shapes must match and start with m")
    npts = int(np.prod(lo.shape[1:])) if lo.dim() > 1 else 1
    out = torch.empty_like(lo)
    _lib.check(_lib.load().edg_riemann_rusanov(C.byref(pde.native()), 1, npts, _lib.ptr(lo), _lib.ptr(hi), int(axis),
                                               int(sign), _lib.ptr(out), _stream()), "riemann_rusanov")
    return out.cpu().numpy() if host else out


def riemann_rusanov_batch(lo, hi, pde: PdeDescriptor, axis, sign=1):
    """(F, m, npts...) face batches along +axis."""
    torch = _torch()
    lo, _ = _dev(lo)
    hi, _ = _dev(hi)
    F_ = lo.shape[0]
    npts = int(np.prod(lo.shape[2:])) if lo.dim() > 2 else 1
    out = torch.empty_like(lo)
    _lib.check(_lib.load().edg_riemann_rusanov(C.byref(pde.native()), F_, npts, _lib.ptr(lo), _lib.ptr(hi), int(axis),
                                               int(sign), _lib.ptr(out), _stream()), "riemann_rusanov")
    return out


# ------------------------------------------------------------- corrector --

def corrector_batch(pde: PdeDescriptor, basis: PolynomialBasis, q_end, trace_f, edges, outcomes=None,
                    side_face=None, nbr=None, trace_q=None, out=None, dt_slots=None, hmin=None, status=None):
    """Corrector of many cells (kernels.py:176-193 per cell).

    Generic: outcomes (F, m, n^(d-1)) + side_face (C, 2d) int32 indices.
    Fused Cartesian: nbr (C, 2d) int32 neighbours (-1 = outflow) + trace_q.
    """
    torch = _torch()
    C_ = q_end.shape[0]
    e, per = _edges_dev(edges, pde.dim, C_)
    if out is None:
        out = torch.empty_like(q_end)
    st = _lib.load().edg_corrector(C.byref(pde.native()), basis.order, _lib.ptr(basis.device_table()), C_,
                                   _lib.ptr(q_end), _lib.ptr(trace_q), _lib.ptr(trace_f), _lib.ptr(nbr),
                                   _lib.ptr(side_face), _lib.ptr(outcomes), _lib.ptr(e), per, _lib.ptr(out),
                                   _lib.ptr(dt_slots), _lib.ptr(hmin), _lib.ptr(status), _stream())
    _lib.check(st, "corrector")
    return out


def corrector(store: PredictorStore, outcomes: dict, basis: PolynomialBasis, edges):
    """Drop-in for kernels.py:176-193."""
    torch = _torch()
    q_end, host = _dev(store.q_end)
    dim = q_end.dim() - 1
    m = q_end.shape[0]
    keys = trace_keys(dim)
    for a, s in keys:
        if (a, s) not in outcomes:
            raise AssertionError(f"face outcome missing for axis {a} side {s}")
    tf = torch.stack([_dev(store.trace_f[k])[0] for k in keys])[None]
    oc = torch.stack([_dev(outcomes[k])[0] for k in keys])
    side = torch.arange(2 * dim, dtype=torch.int32, device="cuda")[None].contiguous()
    pde_stub = PdeDescriptor("euler" if m == dim + 2 else "advection", m, dim, None, None, False,
                             velocity=(0.0,) * dim)
    r = corrector_batch(pde_stub, basis, q_end[None].contiguous(), tf.contiguous(), tuple(edges),
                        outcomes=oc.contiguous(), side_face=side)
    return r[0].cpu().numpy() if host else r[0]


# ------------------------------------------------------------------- FV --

def fv_patch_update_batch(P, pde: PdeDescriptor, dt, edges, halos=None, nbr=None, out=None, dt_slots=None,
                          h_cell=0.0, status=None):
    """FV update of many (B, m, k^d) patches; halos (B, 2d, m, k^(d-1)) or a
    patch neighbour table nbr (B, 2d) (-1 = outflow)."""
    torch = _torch()
    Pd, _ = _dev(P)
    B, m, k = Pd.shape[0], Pd.shape[1], Pd.shape[2]
    if out is None:
        out = torch.empty_like(Pd)
    e = torch.tensor([float(x) for x in edges], dtype=torch.float64, device="cuda") \
        if not isinstance(edges, torch.Tensor) else edges
    dtd = _scalar_dev(dt)
    lib = _lib.load()
    if halos is not None:
        Hd, _ = _dev(halos)
        st = lib.edg_fv_patch_update(C.byref(pde.native()), k, B, _lib.ptr(Pd), _lib.ptr(Hd), _lib.ptr(dtd),
                                     _lib.ptr(e), _lib.ptr(out), _stream())
    else:
        st = lib.edg_fv_patch_step(C.byref(pde.native()), k, B, _lib.ptr(Pd), _lib.ptr(nbr), _lib.ptr(dtd),
                                   _lib.ptr(e), _lib.ptr(out), _lib.ptr(dt_slots), float(h_cell),
                                   _lib.ptr(status), _stream())
    _lib.check(st, "fv_patch_update")
    return out


def fv_patch_update(patch, pde: PdeDescriptor, dt, edges, halos):
    """Drop-in for kernels.py:225-253 (missing halo -> NotReadyError)."""
    torch = _torch()
    Pd, host = _dev(patch)
    dim = Pd.dim() - 1
    for a in range(dim):
        for s in (0, 1):
            if (a, s) not in halos or halos[(a, s)] is None:
                raise NotReadyError(f"halo layer missing for axis {a} side {s}")
    H = torch.stack([_dev(halos[k])[0] for k in trace_keys(dim)])[None]
    r = fv_patch_update_batch(Pd[None], pde, dt, edges, halos=H.contiguous())
    return r[0].cpu().numpy() if host else r[0]


def patch_boundary_layers_batch(P):
    torch = _torch()
    Pd, _ = _dev(P)
    B, m, k = Pd.shape[:3]
    dim = Pd.dim() - 2
    out = torch.empty((B, 2 * dim, m) + (k,) * (dim - 1), dtype=torch.float64, device="cuda")
    _lib.check(_lib.load().edg_patch_boundary_layers(dim, m, k, B, _lib.ptr(Pd), _lib.ptr(out), _stream()),
               "patch_boundary_layers")
    return out


def patch_boundary_layers(patch):
    """Drop-in for kernels.py:256-264."""
    Pd, host = _dev(patch)
    dim = Pd.dim() - 1
    r = patch_boundary_layers_batch(Pd[None])[0]
    return {k: (r[j].cpu().numpy() if host else r[j]) for j, k in enumerate(trace_keys(dim))}


# ------------------------------------------------------------------- dt --

def admissible_dt_device(Q, pde: PdeDescriptor, order, cfl_safety, hmin, dt_out=None, slots=None, status=None):
    """Device-side admissible dt of a (C, m, npts...) batch; returns the
    device scalar (no host sync).  hmin: float or (C,) device tensor."""
    torch = _torch()
    lib = _lib.load()
    Qd, _ = _dev(Q)
    C_, m = Qd.shape[:2]
    npts = int(np.prod(Qd.shape[2:]))
    if slots is None:
        slots = torch.empty(_lib.DT_SLOTS, dtype=torch.int64, device="cuda")
        _lib.check(lib.edg_dt_slots_reset(_lib.ptr(slots), _stream()), "dt reset")
    h = hmin if isinstance(hmin, torch.Tensor) else torch.tensor([float(hmin)], dtype=torch.float64, device="cuda")
    per = 1 if (h.numel() == C_ and C_ > 1) else 0
    _lib.check(lib.edg_cell_speed_reduce(C.byref(pde.native()), int(order), C_, npts, _lib.ptr(Qd), _lib.ptr(h),
                                         per, _lib.ptr(slots), _stream()), "admissible_dt")
    if dt_out is None:
        dt_out = torch.empty(1, dtype=torch.float64, device="cuda")
    if status is None:
        status = torch.zeros(2, dtype=torch.int32, device="cuda")
    _lib.check(lib.edg_dt_finalize(_lib.ptr(slots), float(cfl_safety), _lib.ptr(dt_out), None, 0, _lib.ptr(status),
                                   _stream()), "admissible_dt")
    return dt_out, status


def admissible_dt(cells, pde: PdeDescriptor, order, cfl_safety, mesh):
    """Drop-in for kernels.py:267-281: cells = iterable of (key, q) with
    key[0] the level; mesh provides cell_edges(level)."""
    torch = _torch()
    cells = list(cells)
    if not cells:
        raise EnclaveDgError("no positive wave speed anywhere; cannot pick a time step")
    Q = torch.stack([_dev(q)[0] for _, q in cells])
    h = torch.tensor([min(mesh.cell_edges(k[0])) for k, _ in cells], dtype=torch.float64, device="cuda")
    dt, status = admissible_dt_device(Q, pde, order, cfl_safety, h)
    if int(status[0]) & 1:
        raise EnclaveDgError("no positive wave speed anywhere; cannot pick a time step")
    return float(dt[0])
