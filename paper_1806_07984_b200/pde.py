"""PDE plugins: the reference's PdeDescriptor (pde.py:10-24) carrying, in
addition to its host-side callables, the compile-time specialisation the GPU
kernels use (kind + gamma / velocity).  Python callables cannot cross the C
ABI, so `flux` / `max_eigenvalue` here are only the host-side contract (same
formulas as csrc/edg_common.cuh); the device evaluates its compiled copy.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable

import numpy as np

from . import _lib


@dataclass(frozen=True)
class PdeDescriptor:
    name: str
    m: int
    dim: int
    flux: Callable
    max_eigenvalue: Callable
    is_linear: bool
    gamma: float = 1.4
    velocity: tuple = ()

    def native(self) -> "_lib.EdgPde":
        vel = tuple(self.velocity) + (0.0,) * (3 - len(self.velocity))
        return _lib.make_pde_struct(self.name, self.dim, self.m, self.gamma, vel)


def advection(velocity=(1.0, 0.5), dim: int = 2) -> PdeDescriptor:
    """Scalar linear advection (pde.py:27-37)."""
    a = tuple(float(v) for v in velocity[:dim])

    def flux(q, axis):
        return a[axis] * q

    def max_eig(q, axis):
        return np.full(q.shape[1:], abs(a[axis]))

    return PdeDescriptor("advection", 1, dim, flux, max_eig, True, velocity=a)


def burgers(dim: int = 2) -> PdeDescriptor:
    """Scalar Burgers (pde.py:40-49)."""

    def flux(q, axis):
        return 0.5 * q * q

    def max_eig(q, axis):
        return np.abs(q[0])

    return PdeDescriptor("burgers", 1, dim, flux, max_eig, False)


def euler(dim: int = 2, gamma: float = 1.4) -> PdeDescriptor:
    """Compressible Euler, m = dim + 2 (not in the reference; DESIGN.md
    "Euler plugin" pins the formulas and their operation order)."""
    gm1 = gamma - 1.0

    def _pp(q):
        inv = 1.0 / q[0]
        ke = q[1] * q[1]
        for i in range(1, dim):
            ke = ke + q[1 + i] * q[1 + i]
        ke = 0.5 * ke * inv
        return inv, gm1 * (q[1 + dim] - ke)

    def flux(q, axis):
        inv, p = _pp(q)
        u = q[1 + axis] * inv
        f = np.empty_like(q)
        f[0] = q[1 + axis]
        for i in range(dim):
            f[1 + i] = q[1 + i] * u
        f[1 + axis] = f[1 + axis] + p
        f[1 + dim] = (q[1 + dim] + p) * u
        return f

    def max_eig(q, axis):
        inv, p = _pp(q)
        with np.errstate(invalid="ignore"):
            return np.abs(q[1 + axis] * inv) + np.sqrt(gamma * p * inv)

    return PdeDescriptor("euler", dim + 2, dim, flux, max_eig, False, gamma=gamma)


def make_pde(name: str, dim: int = 2, **kw) -> PdeDescriptor:
    """pde.py:52-57 (+ 'euler')."""
    if name == "advection":
        return advection(dim=dim, **kw)
    if name == "burgers":
        return burgers(dim=dim)
    if name == "euler":
        return euler(dim=dim, **kw)
    raise ValueError(f"unknown pde {name!r}")
