"""ctypes binding of libenclavedg_b200.so (the C ABI in include/enclavedg_b200.h).

This is the reference-side binding a maintainer of the Python reference would
add: plain pointers, sizes and a stream handle.  The library
is loaded from the package's in-tree `_lib/` directory; if it is missing the
import of any compute function fails loudly -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
import re

from .errors import STATUS_ERRORS, NativeError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_lib", "libenclavedg_b200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "enclavedg_b200.h")

PDE_KIND = {"advection": 0, "burgers": 1, "euler": 2}
DT_SLOTS = 256


class EdgPde(C.Structure):
    _fields_ = [("kind", C.c_int32), ("dim", C.c_int32), ("m", C.c_int32), ("reserved", C.c_int32),
                ("gamma", C.c_double), ("velocity", C.c_double * 3)]


P = C.c_void_p
I32 = C.c_int32
D = C.c_double
PDEP = C.POINTER(EdgPde)

SIGNATURES = {
    "edg_supported": (C.c_int, [PDEP, I32]),
    "edg_build_info": (C.c_char_p, []),
    "edg_last_error": (C.c_char_p, []),
    "edg_stp_picard": (C.c_int, [PDEP, I32, P, P, P, I32, P, I32, P, D, I32, P, P, P, P, P, P, P, P]),
    "edg_stp_picard_background": (C.c_int, [PDEP, I32, P, P, P, I32, P, I32, P, D, I32, P, P, P, P, P, P, P, P]),
    "edg_stp_linear": (C.c_int, [PDEP, I32, P, P, P, I32, P, I32, P, P, P, P, P, P, P, P]),
    "edg_probe_fp64": (C.c_int, [P, I32, I32, P]),
    "edg_probe_dmma": (C.c_int, [P, I32, I32, P]),
    "edg_order_by_iterations": (C.c_int, [I32, P, P, P, P]),
    "edg_project_to_faces": (C.c_int, [I32, I32, I32, P, I32, P, P, P]),
    "edg_riemann_rusanov": (C.c_int, [PDEP, I32, I32, P, P, I32, I32, P, P]),
    "edg_corrector": (C.c_int, [PDEP, I32, P, I32, P, P, P, P, P, P, P, I32, P, P, P, P, P]),
    "edg_corrector_grid": (C.c_int, [PDEP, I32, P, I32, I32, P, P, P, P, P, P, P, P, P]),
    "edg_corrector_grid_range": (C.c_int, [PDEP, I32, P, I32, I32, I32, I32, P, P, P, P, P, P, P, P, P]),
    "edg_cell_speed_reduce": (C.c_int, [PDEP, I32, I32, I32, P, P, I32, P, P]),
    "edg_dt_slots_reset": (C.c_int, [P, P]),
    "edg_dt_finalize": (C.c_int, [P, D, P, P, I32, P, P]),
    "edg_faces_rusanov": (C.c_int, [PDEP, I32, P, I32, P, P, P, P, P, P, P]),
    "edg_faces_rusanov_chain": (C.c_int, [PDEP, I32, P, I32, P, P, P, P, P, I32, P, P, P]),
    "edg_faces_restrict": (C.c_int, [I32, I32, I32, P, I32, P, P, P, P, P]),
    "edg_interpolate_face_trace": (C.c_int, [I32, I32, I32, P, I32, P, P, I32, P, P]),
    "edg_fv_patch_update": (C.c_int, [PDEP, I32, I32, P, P, P, P, P, P]),
    "edg_fv_patch_step": (C.c_int, [PDEP, I32, I32, P, P, P, P, P, P, D, P, P]),
    "edg_fv_grid_step": (C.c_int, [PDEP, I32, I32, I32, P, P, P, P, P, D, P, P]),
    "edg_fv_grid_step_range": (C.c_int, [PDEP, I32, I32, I32, I32, I32, P, P, P, P, P, D, P, P]),
    "edg_patch_boundary_layers": (C.c_int, [I32, I32, I32, I32, P, P, P]),
    "edg_stream_priority_range": (C.c_int, [C.POINTER(I32), C.POINTER(I32)]),
    "edg_graph_begin": (C.c_int, [P]),
    "edg_graph_end": (C.c_int, [P, C.POINTER(C.c_void_p), P, I32, C.POINTER(I32)]),
    "edg_graph_launch": (C.c_int, [P, P]),
    "edg_graph_destroy": (C.c_int, [P]),
    "edg_trace_next": (C.c_int, [P]),
    "edg_gradient_indicator": (C.c_int, [I32, I32, I32, P, I32, P, P, D, D, I32, I32, P, P, P]),
    "edg_interpolate_volume": (C.c_int, [I32, I32, I32, P, I32, P, P, P, P, P]),
    "edg_restrict_volume": (C.c_int, [I32, I32, I32, P, I32, P, P, P]),
    "edg_pack_face_traces": (C.c_int, [I32, I32, I32, P, P, P, P, P, P]),
    "edg_unpack_face_traces": (C.c_int, [I32, I32, P, P, P, P]),
    "edg_gather_rows": (C.c_int, [I32, I32, P, P, P, P]),
    "edg_scatter_rows": (C.c_int, [I32, I32, P, P, P, P]),
}

_LIB = None


def header_symbols():
    """Function names declared in include/enclavedg_b200.h."""
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(edg_[a-z0-9_]+)\s*\(", text)))


def load(path: str = LIB_PATH):
    """Load the native library (raises NativeError when it is not built)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(path):
        raise NativeError(f"{path} is missing: run `python -m paper_1806_07984_b200.build_lib` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib


def check(status: int, what: str):
    if status != 0:
        msg = load().edg_last_error().decode(errors="replace")
        raise STATUS_ERRORS.get(status, NativeError)(f"{what}: {msg} (status {status})")


def ptr(t):
    """Raw device pointer of a torch tensor (None -> NULL)."""
    return None if t is None else C.c_void_p(t.data_ptr())


def make_pde_struct(kind: str, dim: int, m: int, gamma: float = 1.4, velocity=(0.0, 0.0, 0.0)) -> EdgPde:
    v = (list(velocity) + [0.0, 0.0, 0.0])[:3]
    return EdgPde(PDE_KIND[kind], dim, m, 0, float(gamma), (C.c_double * 3)(*v))
