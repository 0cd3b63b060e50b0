"""The five BASELINE.json configurations as seeded synthetic inputs.

Pure numpy (no torch, no CUDA): the same generator feeds the GPU solver, the
CPU oracle and the golden-fixture script, so both paths start from identical
bits.  Pinned readings of the prose in BASELINE.json:configs (see DESIGN.md
section "Pinned config readings"):

* cell order is row-major over the Cartesian cell index (axis 0 slowest) for
  uniform meshes; the AMR mesh (config 5) uses the reference's depth-first SFC
  order (mesh.py:322-338);
* node coordinates are x = (cell_index + xi_j) * h with xi_j the GL nodes of
  basis.py:17-25; FV cell centres are (i + 0.5) * h;
* per-node noise is drawn in one `default_rng(seed).uniform` call shaped
  (cells, nodes...) in that cell order;
* "width 0.02" of the blast interface: s = (1 - tanh((r - 0.25) / 0.02)) / 2;
* the seeded centre c of configs 2 and 5 is 0.3 + 0.4 * default_rng(seed).random(2);
* config 5 refines every level-4 cell whose centre satisfies |x - c|^2 < 0.2^2;
* CFL safeties: cfg1 0.9 and cfg2 0.9 as stated; cfg4 0.4 as stated (FV
  dt = cfl * h / max lambda, i.e. admissible_dt with order 0); cfg3 and cfg5
  state none -- pinned to 0.2, the one value verified parity-safe
  (hard part 1).
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass, field, replace

import numpy as np

GAMMA = 1.4


@dataclass(frozen=True)
class Config:
    name: str
    kind: str            # 'dg' (uniform Cartesian), 'dg-amr', 'fv'
    pde: str             # 'advection' | 'euler'
    dim: int
    order: int           # DG polynomial order p (0 for FV)
    cells: int           # cells per axis (uniform) / base cells per axis (AMR) / FV cells per axis
    periodic: bool
    cfl: float
    steps: int
    seed: int = 0
    patch: int = 8       # FV patch edge in cells
    velocity: tuple = (1.0, 0.5)

    @property
    def m(self):
        return 1 if self.pde == "advection" else self.dim + 2

    @property
    def n(self):
        return self.order + 1

    def with_(self, **kw):
        return replace(self, **kw)


CONFIGS = {
    "cfg1": Config("cfg1", "dg", "advection", 2, 3, 27, True, 0.9, 20),
    "cfg2": Config("cfg2", "dg", "euler", 2, 5, 243, True, 0.9, 50),
    "cfg3": Config("cfg3", "dg", "euler", 3, 4, 64, False, 0.2, 20),
    "cfg4": Config("cfg4", "fv", "euler", 3, 0, 128, False, 0.4, 100),
    "cfg5": Config("cfg5", "dg-amr", "euler", 2, 3, 81, True, 0.2, 50),
}


def gl_nodes(n):
    x, _ = np.polynomial.legendre.leggauss(n)
    return 0.5 * (x + 1.0)


def seeded_centre(seed):
    return 0.3 + 0.4 * np.random.default_rng(seed).random(2)


def _node_coords(cell_idx, h, n, dim):
    """(C, dim, n, ..., n) physical node coordinates for cells with integer
    index rows `cell_idx` (C, dim) and edge h (scalar or (C,))."""
    xi = gl_nodes(n)
    C = cell_idx.shape[0]
    h = np.broadcast_to(np.asarray(h, dtype=float), (C,))
    out = np.empty((C, dim) + (n,) * dim)
    for t in range(dim):
        shape = [1] * dim
        shape[t] = n
        loc = xi.reshape(shape)
        out[:, t] = (cell_idx[:, t].reshape((C,) + (1,) * dim) + loc) * h.reshape((C,) + (1,) * dim)
    return out


def uniform_cell_index(N, dim):
    return np.array(list(itertools.product(range(N), repeat=dim)), dtype=np.int64)


def gaussian_bump_state(X, centre):
    """Configs 2/5: rho = 1 + 0.2 exp(-|x - c|^2 / 0.01), u = (1, 1), p = 1."""
    r2 = (X[:, 0] - centre[0]) ** 2 + (X[:, 1] - centre[1]) ** 2
    rho = 1.0 + 0.2 * np.exp(-r2 / 0.01)
    q = np.empty((X.shape[0], 4) + X.shape[2:])
    q[:, 0] = rho
    q[:, 1] = rho * 1.0
    q[:, 2] = rho * 1.0
    q[:, 3] = 1.0 / (GAMMA - 1.0) + 0.5 * rho * 2.0
    return q


def blast_state(X, noise):
    """Configs 3/4: tanh-smoothed spherical blast about the cube centre."""
    r = np.sqrt(sum((X[:, t] - 0.5) ** 2 for t in range(3)))
    s = 0.5 * (1.0 - np.tanh((r - 0.25) / 0.02))
    rho = (0.125 + 0.875 * s) * (1.0 + noise)
    p = 0.1 + 0.9 * s
    q = np.zeros((X.shape[0], 5) + X.shape[2:])
    q[:, 0] = rho
    q[:, 4] = p / (GAMMA - 1.0)
    return q


def initial_dg_uniform(cfg: Config, window=None):
    """(C, m, n^d) initial DoFs of a uniform DG config, row-major cell order.

    window=(lo, size) restricts the output to the size^d block of cells
    starting at cell index (lo,)*d (row-major inside the block); the values
    are exactly those of the full-grid field (noise drawn for the full grid).
    """
    N, d, n = cfg.cells, cfg.dim, cfg.n
    h = 1.0 / N
    idx = uniform_cell_index(N, d)
    sel = slice(None)
    if window is not None:
        lo, size = window
        sel = np.all((idx >= lo) & (idx < lo + size), axis=1)
    X = _node_coords(idx[sel], h, n, d)
    rng = np.random.default_rng(cfg.seed)
    if cfg.pde == "advection":
        noise = rng.uniform(-1e-3, 1e-3, size=(idx.shape[0],) + (n,) * d)[sel]
        u = np.sin(2 * np.pi * X[:, 0]) * np.sin(2 * np.pi * X[:, 1]) + noise
        return u[:, None].copy()
    if d == 2:
        return gaussian_bump_state(X, seeded_centre(cfg.seed))
    noise = rng.uniform(-0.01, 0.01, size=(idx.shape[0],) + (n,) * d)[sel]
    return blast_state(X, noise)


def initial_fv(cfg: Config):
    """(P, 5, k, k, k) patches of the FV config, patches row-major, cells
    row-major inside a patch; noise drawn over the global row-major grid."""
    N, k = cfg.cells, cfg.patch
    h = 1.0 / N
    g = (np.arange(N) + 0.5) * h
    Xg = np.stack(np.meshgrid(g, g, g, indexing="ij"))            # (3, N, N, N)
    noise = np.random.default_rng(cfg.seed).uniform(-0.01, 0.01, size=(N, N, N))
    qg = blast_state(Xg[None], noise[None])[0]                     # (5, N, N, N)
    return grid_to_patches(qg, k)


def grid_to_patches(qg, k):
    m, N = qg.shape[0], qg.shape[1]
    P = N // k
    t = qg.reshape(m, P, k, P, k, P, k).transpose(1, 3, 5, 0, 2, 4, 6)
    return np.ascontiguousarray(t.reshape(P ** 3, m, k, k, k))


def patches_to_grid(patches, k):
    B, m = patches.shape[:2]
    P = round(B ** (1 / 3))
    t = patches.reshape(P, P, P, m, k, k, k).transpose(3, 0, 4, 1, 5, 2, 6)
    return np.ascontiguousarray(t.reshape(m, P * k, P * k, P * k))


def amr_cells(cfg: Config):
    """Real cells (level, index) of config 5's static 2-level mesh (unordered)."""
    L0 = int(round(np.log(cfg.cells) / np.log(3)))
    assert 3 ** L0 == cfg.cells, "AMR base must be a power of 3"
    c = seeded_centre(cfg.seed)
    n0 = cfg.cells
    h = 1.0 / n0
    out = []
    for idx in itertools.product(range(n0), repeat=cfg.dim):
        ctr = [(i + 0.5) * h for i in idx]
        r2 = sum((ctr[t] - c[t]) ** 2 for t in range(cfg.dim))
        if r2 < 0.2 * 0.2:
            for dg in itertools.product(range(3), repeat=cfg.dim):
                out.append((L0 + 1, tuple(3 * i + g for i, g in zip(idx, dg))))
        else:
            out.append((L0, tuple(idx)))
    return out


def sfc_sort(cells, dim):
    """Depth-first 3-tree order with lexicographic child digits (mesh.py:322-338)."""
    def key(cell):
        level, idx = cell
        return tuple(tuple((idx[t] // 3 ** (level - l)) % 3 for t in range(dim))
                     for l in range(1, level + 1))
    return sorted(cells, key=key)


def initial_dg_amr(cfg: Config, cells_sfc):
    """(C, 4, n, n) initial DoFs of config 5 in the given cell order."""
    n = cfg.n
    levels = np.array([l for l, _ in cells_sfc])
    idx = np.array([ix for _, ix in cells_sfc], dtype=np.int64)
    h = 1.0 / 3.0 ** levels
    X = _node_coords(idx, h, n, cfg.dim)
    return gaussian_bump_state(X, seeded_centre(cfg.seed))


def dof_count(cfg: Config, ncells=None):
    if cfg.kind == "fv":
        return cfg.cells ** 3 * cfg.m
    if ncells is None:
        ncells = cfg.cells ** cfg.dim
    return ncells * cfg.m * cfg.n ** cfg.dim
