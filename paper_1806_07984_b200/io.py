"""Solution dump (the SPEC's `dump_solution(mesh,
path)` artifact plumbing, which the reference package does not ship).

CSV columns `level,ix,iy,node_x,node_y,component,value` (3-D adds `iz` and
`node_z`), one row per quadrature-point value of every real cell, in a
stable order: cells in the mesh's storage order (row-major for Cartesian
meshes, the depth-first 3-tree order for adaptive ones), then node index
(C order over the cell's axes), then component.  Values are written with
`repr` (shortest round-trip), so dump -> load -> dump is byte-identical.
"""
from __future__ import annotations

import csv

import numpy as np

from .configs import gl_nodes
from .errors import ConfigError
from .mesh import AdaptiveMesh, CartesianMesh


def _cells(mesh):
    """(levels (C,), integer index (C, d), edge h (C,), dim) of the mesh's cells in storage order."""
    if isinstance(mesh, CartesianMesh):
        return (np.zeros(mesh.ncells, dtype=np.int64), mesh.index.astype(np.int64),
                np.full(mesh.ncells, mesh.h), mesh.dim)
    if isinstance(mesh, AdaptiveMesh):
        lv = np.array([l for l, _ in mesh.cells], dtype=np.int64)
        ix = np.array([i for _, i in mesh.cells], dtype=np.int64)
        return lv, ix, mesh.extent / 3.0 ** lv, mesh.dim
    raise ConfigError(f"dump_solution: unsupported mesh type {type(mesh).__name__}")


def dump_solution(mesh, Q, path) -> int:
    """Write the DoFs `Q` (C, m, n, ..., n) of `mesh` to `path`; returns the row count.

    Raises OSError naming the path on I/O failure (SPEC: "error with path")."""
    Q = np.asarray(Q.cpu() if hasattr(Q, "cpu") else Q, dtype=np.float64)
    lv, ix, h, d = _cells(mesh)
    if Q.ndim != 2 + d or Q.shape[0] != lv.shape[0] or len(set(Q.shape[2:])) != 1:
        raise ConfigError(f"dump_solution: state shape {Q.shape} does not match the mesh ({lv.shape[0]} cells, dim {d})")
    C, m, n = Q.shape[0], Q.shape[1], Q.shape[2]
    xi = gl_nodes(n)
    axes = "xyz"[:d]
    header = ["level"] + [f"i{a}" for a in axes] + [f"node_{a}" for a in axes] + ["component", "value"]
    node_idx = np.array(np.unravel_index(np.arange(n ** d), (n,) * d)).T      # (n^d, d), C order
    flat = Q.reshape(C, m, n ** d)
    rows = 0
    try:
        with open(path, "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(header)
            for c in range(C):
                coords = (ix[c][None, :] + xi[node_idx]) * h[c]            # (n^d, d)
                for p in range(n ** d):
                    pre = [int(lv[c])] + [int(v) for v in ix[c]] + [repr(float(v)) for v in coords[p]]
                    for k in range(m):
                        w.writerow(pre + [k, repr(float(flat[c, k, p]))])
                        rows += 1
    except OSError as e:
        raise OSError(f"dump_solution: cannot write {path}: {e}") from e
    return rows


def load_solution(mesh, path, m=None):
    """Read a dump back into a (C, m, n, ..., n) array in the mesh's cell order."""
    lv, ix, h, d = _cells(mesh)
    C = lv.shape[0]
    with open(path, newline="") as fh:
        r = csv.reader(fh)
        header = next(r)
        vals = [float(row[-1]) for row in r]
    if header[0] != "level" or header[-1] != "value":
        raise ConfigError(f"load_solution: {path} is not a solution dump")
    total = len(vals)
    if m is None:
        with open(path, newline="") as fh:
            r = csv.reader(fh)
            next(r)
            comps = {int(row[-2]) for row in r}
        m = len(comps)
    npts = total // (C * m)
    n = int(round(npts ** (1.0 / d)))
    if C * m * n ** d != total:
        raise ConfigError(f"load_solution: {total} values do not fit {C} cells x {m} components")
    a = np.array(vals).reshape(C, n ** d, m).transpose(0, 2, 1)
    return a.reshape((C, m) + (n,) * d)
