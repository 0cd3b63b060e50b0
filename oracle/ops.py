"""Per-cell numpy restatement of the reference hot-path kernels (oracle only).

Each function names the reference file:line (under
/root/reference/pkg/src/enclavedg/) whose arithmetic it restates.  The numpy
primitives (tensordot contraction axes, operation order) are chosen so that the
results are bit-for-bit those of the reference on the same inputs; this is
pinned by tests/test_oracle_golden.py against tests/golden/*.npz.

Array conventions (reference kernels.py:5-10): component axis first, then one
axis of n = p + 1 Gauss-Legendre nodes per space dimension in x, y[, z] order;
a face trace drops the face-normal axis; traces are time-integrated.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable

import numpy as np

MAX_NODES = 16          # basis.py:13
ORDERS = (1, 7)         # basis.py:14


class OracleConfigError(ValueError):
    """Order / node count out of range (reference errors.ConfigError)."""


class OracleNotReady(RuntimeError):
    """Missing halo / incomplete parent (reference errors.NotReadyError)."""


class OracleNoWaveSpeed(RuntimeError):
    """No positive wave speed (reference kernels.py:279-280)."""


# ---------------------------------------------------------------- basis ---

def gl_rule(n: int):
    """n-point Gauss-Legendre rule mapped to [0, 1] (basis.py:17-25)."""
    if n < 1 or n > MAX_NODES:
        raise OracleConfigError(f"quadrature point count {n} outside [1, {MAX_NODES}]")
    x, w = np.polynomial.legendre.leggauss(n)
    return 0.5 * (x + 1.0), 0.5 * w


class Basis:
    """Nodal Lagrange basis on GL points of [0,1] (basis.py:34-85).

    Attributes mirror the reference: order, n, nodes, weights, diff_matrix
    (D[i, j] = l_j'(x_i)), trace_left / trace_right (l_j(0), l_j(1)).
    """

    def __init__(self, order: int):
        if not ORDERS[0] <= order <= ORDERS[1]:
            raise OracleConfigError(f"polynomial order {order} outside {ORDERS}")
        self.order = order
        self.n = order + 1
        self.nodes, self.weights = gl_rule(self.n)
        gap = self.nodes[:, None] - self.nodes[None, :]          # basis.py:28-31
        np.fill_diagonal(gap, 1.0)
        self.bary = 1.0 / gap.prod(axis=1)
        self.diff_matrix = self._derivative()
        self.trace_left = self.lagrange_eval(np.array([0.0]))[0]
        self.trace_right = self.lagrange_eval(np.array([1.0]))[0]

    def _derivative(self):
        """basis.py:57-65 (off-diagonal barycentric formula, negative row sum)."""
        x, b, n = self.nodes, self.bary, self.n
        dm = np.zeros((n, n))
        for i in range(n):
            for j in range(n):
                if j != i:
                    dm[i, j] = (b[j] / b[i]) / (x[i] - x[j])
            dm[i, i] = -dm[i].sum()
        return dm

    def lagrange_eval(self, points):
        """E[k, j] = l_j(points[k]) (basis.py:67-81)."""
        pts = np.asarray(points, dtype=float)
        table = np.empty((len(pts), self.n))
        for k, x in enumerate(pts):
            d = x - self.nodes
            hit = np.isclose(d, 0.0, atol=1e-14)
            if hit.any():
                row = np.zeros(self.n)
                row[np.argmax(hit)] = 1.0
            else:
                row = self.bary / d
                row /= row.sum()
            table[k] = row
        return table

    def trace(self, side: int):
        return self.trace_left if side == 0 else self.trace_right


_BASES: dict = {}


def basis_for(order: int) -> Basis:
    """Cached basis (basis.py:88-94)."""
    if order not in _BASES:
        _BASES[order] = Basis(order)
    return _BASES[order]


_KINV: dict = {}


def time_operators(basis: Basis):
    """K^-1 of the weak-in-time collocation matrix and the lift (kernels.py:109-117)."""
    if basis.order not in _KINV:
        kmat = np.outer(basis.trace_right, basis.trace_right)
        kmat -= basis.diff_matrix.T * basis.weights[None, :]
        _KINV[basis.order] = (np.linalg.inv(kmat), basis.trace_left.copy())
    return _KINV[basis.order]


# ------------------------------------------------------------------ PDEs ---

@dataclass(frozen=True)
class Pde:
    """Reference PdeDescriptor plugin (pde.py:10-24) plus the parameters the
    GPU build needs to specialise flux / wave speed at compile time."""

    name: str
    m: int
    dim: int
    flux: Callable
    max_eigenvalue: Callable
    is_linear: bool
    gamma: float = 1.4
    velocity: tuple = ()


def advection(velocity=(1.0, 0.5), dim=2) -> Pde:
    """pde.py:27-37."""
    a = tuple(float(v) for v in velocity[:dim])

    def flux(q, axis):
        return a[axis] * q

    def lam(q, axis):
        return np.full(q.shape[1:], abs(a[axis]))

    return Pde("advection", 1, dim, flux, lam, True, velocity=a)


def burgers(dim=2) -> Pde:
    """pde.py:40-49."""

    def flux(q, axis):
        return 0.5 * q * q

    def lam(q, axis):
        return np.abs(q[0])

    return Pde("burgers", 1, dim, flux, lam, False)


def _euler_parts(q, dim, gm1):
    """Shared primitive quantities of the Euler system (oracle-defined, see
    DESIGN.md "Euler plugin"): 1/rho, kinetic energy density, pressure."""
    inv = 1.0 / q[0]
    ke = q[1] * q[1]
    for i in range(1, dim):
        ke = ke + q[1 + i] * q[1 + i]
    ke = 0.5 * ke * inv
    p = gm1 * (q[1 + dim] - ke)
    return inv, p


def euler(dim=2, gamma=1.4) -> Pde:
    """Compressible Euler, m = dim + 2, added in the reference plugin format
    (pde.py:10-24); the reference ships none.

    flux_a = (rho u_a, rho u_i u_a + delta_ia p, (E + p) u_a),
    lambda_a = |u_a| + sqrt(gamma p / rho), p = (gamma - 1)(E - |rho u|^2 / (2 rho)).
    The operation order below is the contract the CUDA flux mirrors.
    """
    gm1 = gamma - 1.0

    def flux(q, axis):
        inv, p = _euler_parts(q, dim, gm1)
        u = q[1 + axis] * inv
        out = np.empty_like(q)
        out[0] = q[1 + axis]
        for i in range(dim):
            out[1 + i] = q[1 + i] * u
        out[1 + axis] = out[1 + axis] + p
        out[1 + dim] = (q[1 + dim] + p) * u
        return out

    def lam(q, axis):
        inv, p = _euler_parts(q, dim, gm1)
        u = q[1 + axis] * inv
        with np.errstate(invalid="ignore"):
            c = np.sqrt(gamma * p * inv)
        return np.abs(u) + c

    return Pde("euler", dim + 2, dim, flux, lam, False, gamma=gamma)


def make_pde(name, dim=2, **kw) -> Pde:
    """pde.py:52-57 (+ 'euler')."""
    if name == "advection":
        return advection(dim=dim, **kw)
    if name == "burgers":
        return burgers(dim=dim)
    if name == "euler":
        return euler(dim=dim, **kw)
    raise ValueError(f"unknown pde {name!r}")


# --------------------------------------------------------------- kernels ---

@dataclass
class Store:
    """PredictorStore (kernels.py:25-41)."""

    q_int: np.ndarray
    q_end: np.ndarray
    trace_q: dict
    trace_f: dict
    iterations: int = 0
    converged: bool = True


def nodal_divergence(q, pde, basis, edges):
    """sum_a D (x) F_a(q) / h_a along axis a (kernels.py:63-70)."""
    acc = np.zeros_like(q)
    for a in range(q.ndim - 1):
        fa = pde.flux(q, a)
        acc += np.moveaxis(np.tensordot(basis.diff_matrix, fa, axes=(1, 1 + a)), 0, 1 + a) / edges[a]
    return acc


def face_traces(vol, basis):
    """Extrapolate volume data to the 2d faces (kernels.py:73-79)."""
    d = vol.ndim - 1
    return {(a, s): np.tensordot(basis.trace(s), vol, axes=(0, 1 + a))
            for a in range(d) for s in (0, 1)}


def predictor_ck(q, pde, dt, basis, edges) -> Store:
    """Cauchy-Kowalevski predictor for linear PDEs (kernels.py:82-106)."""
    if not pde.is_linear:
        raise ValueError("stp_linear requires a linear flux")
    d = q.ndim - 1
    q_end = q.copy()
    q_int = dt * q
    term = q
    fact = 1.0
    for k in range(1, d * basis.order + 1):
        term = -nodal_divergence(term, pde, basis, edges)
        fact *= k
        q_end += (dt ** k / fact) * term
        q_int += (dt ** (k + 1) / (fact * (k + 1))) * term
    tq = face_traces(q_int, basis)
    tf = {key: pde.flux(v, key[0]) for key, v in tq.items()}
    return Store(q_int, q_end, tq, tf)


def predictor_picard(q, pde, dt, basis, edges, tol=1e-10, max_iter=None) -> Store:
    """Weak-in-time Picard space-time predictor (kernels.py:120-159)."""
    if max_iter is None:
        max_iter = 2 * basis.n
    kinv, lift = time_operators(basis)
    nt = basis.n
    w = basis.weights
    qhat = np.repeat(q[None], nt, axis=0)
    base = np.tensordot(kinv @ lift[:, None], q[None], axes=(1, 0))
    its, done = 0, False
    for it in range(1, max_iter + 1):
        its = it
        rhs = np.stack([-dt * w[r] * nodal_divergence(qhat[r], pde, basis, edges) for r in range(nt)])
        nxt = base + np.tensordot(kinv, rhs, axes=(1, 0))
        delta = float(np.abs(nxt - qhat).max())
        qhat = nxt
        if delta < tol:
            done = True
            break
    return _predictor_epilogue(q.ndim - 1, qhat, pde, dt, basis, its, done)


def _predictor_epilogue(d, qhat, pde, dt, basis, its, done):
    """End state, time integral and the two trace families (kernels.py:148-159)."""
    w = basis.weights
    q_end = np.tensordot(basis.trace_right, qhat, axes=(0, 0))
    q_int = dt * np.tensordot(w, qhat, axes=(0, 0))
    tq = face_traces(q_int, basis)
    tf = {}
    for a in range(d):
        fn = np.stack([pde.flux(qhat[r], a) for r in range(basis.n)])
        fi = dt * np.tensordot(w, fn, axes=(0, 0))
        for s in (0, 1):
            tf[(a, s)] = np.tensordot(basis.trace(s), fi, axes=(0, 1 + a))
    return Store(q_int, q_end, tq, tf, iterations=its, converged=done)


def rusanov(lo, hi, pde, axis, sign=1):
    """Pointwise Rusanov flux along +axis (kernels.py:162-173)."""
    lam = np.maximum(pde.max_eigenvalue(lo, axis), pde.max_eigenvalue(hi, axis))
    central = 0.5 * (pde.flux(lo, axis) + pde.flux(hi, axis))
    jump = 0.5 * lam * (hi - lo)
    if sign >= 0:
        return central - jump
    return -central + jump


def correct(store: Store, outcomes: dict, basis, edges):
    """Predictor end state minus the surface jump terms (kernels.py:176-193)."""
    q = store.q_end.copy()
    for a in range(q.ndim - 1):
        for s in (0, 1):
            if (a, s) not in outcomes:
                raise AssertionError(f"face outcome missing for axis {a} side {s}")
            jump = outcomes[(a, s)] - store.trace_f[(a, s)]
            sgn = 1.0 if s == 1 else -1.0
            lift = sgn * basis.trace(s) / (basis.weights * edges[a])
            q -= np.moveaxis(np.tensordot(lift, jump, axes=0), 0, 1 + a)
    return q


def fv_update(patch, pde, dt, edges, halos):
    """Unsplit first-order Rusanov update of a k^d patch (kernels.py:225-253)."""
    d = patch.ndim - 1
    k = patch.shape[1]
    for a in range(d):
        for s in (0, 1):
            if halos.get((a, s)) is None:
                raise OracleNotReady(f"halo layer missing for axis {a} side {s}")
    out = patch.copy()
    for a in range(d):
        dx = edges[a] / k
        ext = np.concatenate([np.expand_dims(halos[(a, 0)], 1 + a), patch,
                              np.expand_dims(halos[(a, 1)], 1 + a)], axis=1 + a)
        ext = np.moveaxis(ext, 1 + a, 1)
        fl = [rusanov(ext[:, i], ext[:, i + 1], pde, a) for i in range(k + 1)]
        view = np.moveaxis(out, 1 + a, 1)
        for i in range(k):
            view[:, i] -= (dt / dx) * (fl[i + 1] - fl[i])
    return out


def boundary_layers(patch):
    """Outermost layers keyed (axis, side) (kernels.py:256-264)."""
    out = {}
    for a in range(patch.ndim - 1):
        mv = np.moveaxis(patch, 1 + a, 1)
        out[(a, 0)] = mv[:, 0].copy()
        out[(a, 1)] = mv[:, -1].copy()
    return out


def cell_speed(q, pde, dim):
    """Per-cell lambda of admissible_dt (kernels.py:271-273): Python max over
    axes of the numpy max over nodes -- NaN axes are dropped by Python max."""
    lam = 0.0
    for a in range(dim):
        lam = max(lam, float(pde.max_eigenvalue(q, a).max()))
    return lam


def stable_dt(cells, pde, order, cfl, dim):
    """Global step (kernels.py:267-281).  cells: iterable of (h_min, q)."""
    best = None
    for h, q in cells:
        lam = cell_speed(q, pde, dim)
        if lam <= 0.0:
            continue
        cand = h / ((2 * order + 1) * lam)
        best = cand if best is None else min(best, cand)
    if best is None:
        raise OracleNoWaveSpeed("no positive wave speed anywhere; cannot pick a time step")
    return cfl * best
