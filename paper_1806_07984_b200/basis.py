"""Host-side nodal basis (Gauss-Legendre on [0,1]) and the packed operator
table uploaded to the GPU.

Same API as the reference basis module (/root/reference/pkg/src/enclavedg/
basis.py:17-94): gauss_legendre, PolynomialBasis, get_basis.  The operators
are computed with numpy in the reference's own way (so the uploaded bits are
the reference's; pinned by tests/test_host.py against tests/golden/ops.npz)
and then never recomputed on the device.  The time operators follow
kernels.py:109-114, the 3:1 transfer matrices transfer.py:28-39.
"""
from __future__ import annotations

import numpy as np

from .errors import ConfigError

MAX_QUADRATURE_POINTS = 16
ORDER_RANGE = (1, 7)


def gauss_legendre(n: int):
    """Nodes and weights of the n-point GL rule on [0, 1] (basis.py:17-25)."""
    if not 1 <= n <= MAX_QUADRATURE_POINTS:
        raise ConfigError(f"quadrature point count {n} outside [1, {MAX_QUADRATURE_POINTS}]")
    x, w = np.polynomial.legendre.leggauss(n)
    return 0.5 * (x + 1.0), 0.5 * w


class PolynomialBasis:
    """Degree-p nodal Lagrange basis on GL points (basis.py:34-85)."""

    def __init__(self, order: int):
        lo, hi = ORDER_RANGE
        if not lo <= order <= hi:
            raise ConfigError(f"polynomial order {order} outside [{lo}, {hi}]")
        self.order = order
        self.n = order + 1
        self.nodes, self.weights = gauss_legendre(self.n)
        dif = self.nodes[:, None] - self.nodes[None, :]
        np.fill_diagonal(dif, 1.0)
        self._bary = 1.0 / dif.prod(axis=1)
        self.diff_matrix = self._diff()
        self.trace_left = self.lagrange_eval(np.array([0.0]))[0]
        self.trace_right = self.lagrange_eval(np.array([1.0]))[0]
        self._tables = {}

    def _diff(self):
        x, b, n = self.nodes, self._bary, self.n
        out = np.zeros((n, n))
        for i in range(n):
            for j in range(n):
                if i != j:
                    out[i, j] = (b[j] / b[i]) / (x[i] - x[j])
            out[i, i] = -out[i].sum()
        return out

    def lagrange_eval(self, points):
        """E[k, j] = l_j(points[k]); exact node hits return unit rows."""
        pts = np.asarray(points, dtype=float)
        out = np.empty((len(pts), self.n))
        for k, x in enumerate(pts):
            d = x - self.nodes
            hit = np.isclose(d, 0.0, atol=1e-14)
            if hit.any():
                row = np.zeros(self.n)
                row[np.argmax(hit)] = 1.0
            else:
                row = self._bary / d
                row /= row.sum()
            out[k] = row
        return out

    def trace(self, side: int):
        return self.trace_left if side == 0 else self.trace_right

    # ---- operators beyond the reference basis, host-computed once -------
    def time_operators(self):
        """(K^-1, lift) of the weak-in-time collocation system (kernels.py:109-114)."""
        k = np.outer(self.trace_right, self.trace_right)
        k -= self.diff_matrix.T * self.weights[None, :]
        return np.linalg.inv(k), self.trace_left.copy()

    def transfer_matrices(self):
        """interp[j], restrict[j] for the three thirds (transfer.py:28-39)."""
        w = self.weights
        interp, restr = [], []
        for j in range(3):
            e = self.lagrange_eval((j + self.nodes) / 3.0)
            interp.append(e)
            restr.append((e.T * w[None, :]) / w[:, None] / 3.0)
        return np.stack(interp), np.stack(restr)

    def packed_table(self) -> np.ndarray:
        """fp64 table in the EDG_BASIS_* layout of include/enclavedg_b200.h."""
        kinv, lift = self.time_operators()
        interp, restr = self.transfer_matrices()
        parts = [self.diff_matrix.ravel(), self.weights, self.trace_left, self.trace_right,
                 kinv.ravel(), (kinv @ lift[:, None]).ravel(), interp.ravel(), restr.ravel()]
        tab = np.concatenate(parts)
        assert tab.size == 8 * self.n ** 2 + 4 * self.n
        return tab

    def device_table(self, device="cuda"):
        """The packed table as a device tensor (cached per device)."""
        import torch
        key = str(device)
        if key not in self._tables:
            self._tables[key] = torch.from_numpy(self.packed_table()).to(device)
        return self._tables[key]


_BASIS_CACHE: dict = {}


def get_basis(order: int) -> PolynomialBasis:
    if order not in _BASIS_CACHE:
        _BASIS_CACHE[order] = PolynomialBasis(order)
    return _BASIS_CACHE[order]
