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


# ------------------------------------------------------------ event logs --

def entity_id(kind, obj):
    """Entity ids in the reference's format (mesh.py:687-690): cells
    'c{level}:{i}:{j}[:{k}]', faces 'f{id}'."""
    if kind == "face":
        return f"f{int(obj)}"
    level, index = obj
    return f"c{int(level)}:" + ":".join(str(int(i)) for i in index)


def dump_event_log(rows, path):
    """Write events as CSV `sweep,kind,entity_id,order_index` -- the
    reference's dump_event_log (mesh.py:679-684), same columns and format."""
    try:
        with open(path, "w") as fh:
            fh.write("sweep,kind,entity_id,order_index\n")
            for sweep, kind, entity, idx in rows:
                fh.write(f"{sweep},{kind},{entity},{idx}\n")
    except OSError as e:
        raise OSError(f"dump_event_log: cannot write {path}: {e}") from e


def schedule_events(mesh, sweep=0):
    """The device schedule's issue order for one step as event rows
    (sweep, kind, entity_id, order_index): on an adaptive mesh the skeleton
    cells' predictors, the skeleton-only leaf faces (every hanging face among
    them), the enclave cells' predictors, then the remaining leaf faces; on a
    Cartesian mesh the cells in storage order (the solver reorders them by
    their last Picard count on the device) and the faces per axis.  This
    replaces the reference's traversal orders (mesh.py:505-628), which have
    no device counterpart."""
    rows = []
    if isinstance(mesh, AdaptiveMesh):
        seq = [("cell", mesh.cells[c]) for c in mesh.skeleton]
        seq += [("face", f) for f in range(mesh.nleaf_skeleton)]
        seq += [("cell", mesh.cells[c]) for c in mesh.enclave]
        seq += [("face", f) for f in range(mesh.nleaf_skeleton, mesh.nleaf)]
    elif isinstance(mesh, CartesianMesh):
        seq = [("cell", (0, tuple(ix))) for ix in mesh.index]
        seq += [("face", f) for f in range(mesh.ncells * mesh.dim)]
    else:
        raise ConfigError(f"schedule_events: unsupported mesh type {type(mesh).__name__}")
    for i, (kind, obj) in enumerate(seq):
        rows.append((sweep, kind, entity_id(kind, obj), i))
    return rows


def dump_trace(records, path, t0=None):
    """Write launch-trace records (solver.LaunchTrace.records()) as the SPEC's
    trace CSV `t_ns,worker,event,entity,sweep`: one `start` and
    one `finish` row per launch (first-CTA start / last-CTA exit on the device
    clock, ns relative to the earliest start), worker = the stream class
    (main / hi / lo), entity = the task kind, rows in time order."""
    if not records:
        rows = []
    else:
        base = min(r[3] for r in records) if t0 is None else t0
        rows = []
        for entity, worker, sweep, start, end in records:
            rows.append((start - base, worker, "start", entity, sweep))
            rows.append((end - base, worker, "finish", entity, sweep))
        rows.sort(key=lambda r: (r[0], r[2] != "finish"))
    try:
        with open(path, "w") as fh:
            fh.write("t_ns,worker,event,entity,sweep\n")
            for r in rows:
                fh.write(f"{r[0]},{r[1]},{r[2]},{r[3]},{r[4]}\n")
    except OSError as e:
        raise OSError(f"dump_trace: cannot write {path}: {e}") from e
    return len(rows)
