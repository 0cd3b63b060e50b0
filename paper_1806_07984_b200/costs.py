"""Algorithmic flop / byte counts per unit of work.

Convention: add/sub/mul/div/sqrt = 1 flop, FMA = 2, abs/max = 0.  Bytes are
compulsory HBM traffic (each operand read once, each result written once).
These are the numerators of the roofline fractions bench.py reports; the
kernels' actual counts are equal or larger (e.g. the reciprocal and the
folded constants), so the fractions are conservative.
"""
from __future__ import annotations


def flux_flops(pde: str, d: int) -> int:
    """Phi: flux of all d axes at one point."""
    if pde == "euler":
        return (2 * d + 5) + d * (d + 3)
    if pde == "burgers":
        return 2 * d
    return d


def stp_iter_flops(pde, d, n, m):
    """One Picard iteration of one cell."""
    return n ** (d + 1) * flux_flops(pde, d) + 2 * (d + 1) * m * n ** (d + 2) + (d + 2) * m * n ** (d + 1)


def stp_iter1_flops(pde, d, n, m):
    """First Picard iteration as the kernel executes it: qhat_s = q for every
    time node, so one flux + one derivative per node and a rank-1 time
    update (acc[r] = c_r q + (sum_s B[r][s]) div F(q))."""
    return n ** d * flux_flops(pde, d) + 2 * d * m * n ** (d + 1) + 3 * m * n ** (d + 1)


def stp_executed_flops(pde, d, n, m, cell_iterations, cell_steps):
    """Flops the kernel executes for `cell_iterations` Picard iterations
    summed over `cell_steps` cell-predictor evaluations."""
    return (cell_steps * (stp_iter1_flops(pde, d, n, m) + stp_epilogue_flops(pde, d, n, m))
            + (cell_iterations - cell_steps) * stp_iter_flops(pde, d, n, m))


def stp_epilogue_flops(pde, d, n, m):
    return (4 * m * n ** (d + 1) + m * n ** d + 8 * d * m * n ** d + n ** (d + 1) * flux_flops(pde, d)
            + 2 * d * m * n ** (d + 1))


def stp_bytes(d, n, m):
    """q in, q_end out, 2d trace_q + 2d trace_f out."""
    return 8 * m * (2 * n ** d + 4 * d * n ** (d - 1))


def riemann_flops(pde, d, n, m):
    lam = 4 if pde == "euler" else 0
    fl = (2 * d + 5 + d + 3) if pde == "euler" else (2 if pde == "burgers" else 1)
    return n ** (d - 1) * (2 * fl + 2 * lam + 1 + 5 * m)


def corrector_flops(pde, d, n, m, fused=True):
    f = 2 * d * m * n ** (d - 1) + 4 * d * m * n ** d
    if fused:
        f += d * riemann_flops(pde, d, n, m)     # one solve per face, d faces per cell
    return f


def corrector_bytes(d, n, m):
    """q_end in, Q out, own trace_q + trace_f in (neighbour traces are the same array)."""
    return 8 * (2 * m * n ** d + 4 * d * m * n ** (d - 1))


def fv_cell_flops(pde, d=3):
    return 274 if (pde == "euler" and d == 3) else 30 * d


def fv_cell_bytes(m):
    return 16 * m
