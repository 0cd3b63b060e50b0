"""Algorithm-1 three-loop time-step drivers (oracle only).

The reference ships no driver; these follow the
paper's Algorithm 1 / SPEC run_oracle
exactly as SURVEY.md section 3(A) lays it out:

    dt = admissible_dt(...)                       kernels.py:267-281
    for cell: store = stp_picard(q, ...)          kernels.py:120-159
    for leaf face: outcome = riemann_rusanov(lo.trace_q[(a,1)], hi.trace_q[(a,0)])
                   [virtual side: interpolate_to_virtual(coarse.trace_q[(a,1-s)], child_pos)]
                   [child face: restrict_riemann into the parent]   transfer.py:75-96
    for cell: q = corrector(store, outcomes, ...) kernels.py:176-193

Outflow boundary ("copy/outflow"): the ghost state is the cell's
own trace (DG) / own boundary layer (FV).

All drivers return (Q_final, log) where log holds per-step dt and per-cell
Picard iteration counts.
"""
from __future__ import annotations

import numpy as np

from . import ops, batched
from .transfer import transfer_for, to_virtual, ParentAccumulator, accumulate_restriction


# ----------------------------------------------------------- uniform DG ---

def _grid(arr, N, dim):
    return arr.reshape((N,) * dim + arr.shape[1:])


def uniform_outcomes(tq, pde, N, dim, periodic):
    """Rusanov outcomes on a Cartesian grid for every cell side.

    tq: {(a, s): (C, m, ...)} time-integrated traces, C = N^dim row-major.
    Face between cell c (lo) and c + e_a (hi) is solved once, along +a.
    """
    out = {}
    for a in range(dim):
        lo = _grid(tq[(a, 1)], N, dim)
        hi = np.roll(_grid(tq[(a, 0)], N, dim), -1, axis=a)
        if not periodic:
            last = [slice(None)] * dim
            last[a] = N - 1
            hi = hi.copy()
            hi[tuple(last)] = lo[tuple(last)]                  # outflow ghost = own trace
        C = N ** dim
        up = batched.rusanov_b(lo.reshape((C,) + lo.shape[dim:]),
                               hi.reshape((C,) + hi.shape[dim:]), pde, a)
        down = np.roll(_grid(up, N, dim), 1, axis=a)
        if not periodic:
            first = [slice(None)] * dim
            first[a] = 0
            own = _grid(tq[(a, 0)], N, dim)[tuple(first)]
            own_c = own.reshape((-1,) + own.shape[dim - 1:])
            down = down.copy()
            bnd = batched.rusanov_b(own_c, own_c, pde, a)
            down[tuple(first)] = bnd.reshape(own.shape)
        out[(a, 1)] = up
        out[(a, 0)] = down.reshape(up.shape)
    return out


def dg_uniform_step(Q, pde, basis, N, dim, periodic, cfl, dt=None, h=None):
    """One Algorithm-1 step on a uniform N^dim grid with batched kernels
    (cell edge h, default 1/N)."""
    h = 1.0 / N if h is None else h
    edges = (h,) * dim
    if dt is None:
        dt = batched.stable_dt_b(Q, h, pde, basis.order, cfl, dim)
    st = batched.predictor_picard_b(Q, pde, dt, basis, edges)
    outc = uniform_outcomes(st["trace_q"], pde, N, dim, periodic)
    Qn = batched.correct_b(st["q_end"], st["trace_f"], outc, basis, edges)
    return Qn, dt, st


def dg_uniform_run(Q0, pde, order, N, dim, periodic, cfl, steps, on_step=None, h=None):
    basis = ops.basis_for(order)
    Q = Q0.copy()
    log = {"dt": [], "iterations": []}
    for k in range(steps):
        Q, dt, st = dg_uniform_step(Q, pde, basis, N, dim, periodic, cfl, h=h)
        log["dt"].append(dt)
        log["iterations"].append(st["iterations"].copy())
        if on_step is not None:
            on_step(k, Q)
    return Q, log


def dg_uniform_step_percell(Q, pde, basis, N, dim, periodic, cfl, dt=None, cells=None, h=None):
    """Per-cell reference structure (one stp_picard call per cell); `cells`
    restricts the predictor and corrector loops to a subset (CPU-baseline
    sampling), in which case the returned Q is only valid on that subset."""
    h = 1.0 / N if h is None else h
    edges = (h,) * dim
    C = Q.shape[0]
    if dt is None:
        dt = ops.stable_dt(((h, Q[c]) for c in range(C)), pde, basis.order, cfl, dim)
    sel = range(C) if cells is None else cells
    stores = {c: ops.predictor_picard(Q[c], pde, dt, basis, edges) for c in sel}
    strides = [N ** (dim - 1 - t) for t in range(dim)]
    Qn = Q.copy()
    for c in sel:
        idx = [(c // strides[t]) % N for t in range(dim)]
        res = {}
        for a in range(dim):
            for s in (0, 1):
                j = idx[a] + (1 if s else -1)
                if 0 <= j < N or periodic:
                    nb = c + ((j % N) - idx[a]) * strides[a]
                    other = stores.get(nb)
                    if other is None:       # sampled run: neighbour outside the sample
                        other = stores[c]
                    mine = stores[c].trace_q[(a, s)]
                    theirs = other.trace_q[(a, 1 - s)]
                    lo, hi = (mine, theirs) if s == 1 else (theirs, mine)
                else:
                    lo = hi = stores[c].trace_q[(a, s)]
                res[(a, s)] = ops.rusanov(lo, hi, pde, a)
        Qn[c] = ops.correct(stores[c], res, basis, edges)
    return Qn, dt, stores


# --------------------------------------------------------------- AMR DG ---

def virtual_path(f):
    """Digit tuples from the coarse owner's side face down to leaf face f
    (outermost level last): a virtual side's trace is the owner's trace
    interpolated one level at a time along this path (transfer.py:75-79
    applied level by level -- the multi-level chains of mesh.py:67-100)."""
    owner_level = min(f.owners[s][0] for s in (0, 1) if f.sides[s] == "virtual")
    path, g = [], f
    while g.level > owner_level:
        path.append(g.child_pos)
        g = g.parent
    return path[::-1]


def amr_face_outcomes(forest, stores, pde, ops_t, sweep):
    """Leaf-face Rusanov outcomes and the parent outcomes restricted from
    them (restrict_riemann, transfer.py:82-96), deepest parents first so that
    a parent of a parent accumulates complete children.  With at most one
    level between neighbours this is exactly the one-level scheme."""
    outcome, acc = {}, {}
    for f in forest.leaf_faces():
        a = f.axis
        side_tr = [None, None]
        for s in (0, 1):
            tag = f.sides[s]
            if tag == "cell":
                side_tr[s] = stores[f.owners[s]].trace_q[(a, 1 - s)]
            elif tag == "virtual":
                t = stores[f.owners[s]].trace_q[(a, 1 - s)]
                for digits in virtual_path(f):
                    t = to_virtual(ops_t, t, digits)
                side_tr[s] = t
        if f.sides[0] == "boundary":
            side_tr[0] = side_tr[1]
        if f.sides[1] == "boundary":
            side_tr[1] = side_tr[0]
        out = ops.rusanov(side_tr[0], side_tr[1], pde, a)
        if f.parent is not None:
            buf = acc.setdefault(f.parent.key, ParentAccumulator())
            accumulate_restriction(ops_t, buf, out, f.child_pos, sweep)
        outcome[f.key] = out
    # parents, deepest level first; a parent with a parent restricts into it
    for key in sorted(acc, key=lambda k: -k[1]):
        outcome[key] = acc[key].outcome
        par = forest.faces[key].parent
        if par is not None:
            buf = acc.setdefault(par.key, ParentAccumulator())
            accumulate_restriction(ops_t, buf, outcome[key], forest.faces[key].child_pos, sweep)
    return outcome


def dg_amr_step(forest, Q, pde, basis, cfl, sweep=0, dt=None):
    """One Algorithm-1 step on a static adaptive mesh (per-cell kernels).

    forest: oracle.spacetree.FaceForest; Q: {cell_key: (m, n^d)}.
    """
    dim = forest.dim
    ops_t = transfer_for(basis.order)
    if dt is None:
        dt = ops.stable_dt(((min(forest.cell_edges(k[0])), Q[k]) for k in forest.sfc),
                           pde, basis.order, cfl, dim)
    stores = {k: ops.predictor_picard(Q[k], pde, dt, basis, forest.cell_edges(k[0]))
              for k in forest.sfc}
    outcome = amr_face_outcomes(forest, stores, pde, ops_t, sweep)
    Qn = {}
    for k in forest.sfc:
        res = {(a, s): outcome[forest.side_face_key(k, a, s)] for a in range(dim) for s in (0, 1)}
        Qn[k] = ops.correct(stores[k], res, basis, forest.cell_edges(k[0]))
    return Qn, dt, stores


def dg_amr_run(forest, Q0, pde, order, cfl, steps):
    basis = ops.basis_for(order)
    Q = dict(Q0)
    log = {"dt": [], "iterations": []}
    for k in range(steps):
        Q, dt, st = dg_amr_step(forest, Q, pde, basis, cfl, sweep=k)
        log["dt"].append(dt)
        log["iterations"].append(np.array([st[c].iterations for c in forest.sfc]))
    return Q, log


# ------------------------------------------------------------------- FV ---

def fv_halos(P, dim=3):
    """Halo layers of every patch from its face neighbours' boundary layers
    (kernels.py:256-264); outflow = own boundary layer.  P: (B, m, k, ...)
    with B = np^dim patches row-major."""
    B = P.shape[0]
    npx = round(B ** (1.0 / dim))
    G = P.reshape((npx,) * dim + P.shape[1:])
    halos = {}
    for a in range(dim):
        first = np.take(G, 0, axis=dim + 1 + a)           # (np.., m, k^(d-1)) layer 0
        last = np.take(G, -1, axis=dim + 1 + a)
        lo = np.roll(last, 1, axis=a)                      # neighbour below: its last layer
        hi = np.roll(first, -1, axis=a)
        sl0 = [slice(None)] * dim
        sl0[a] = 0
        sl1 = [slice(None)] * dim
        sl1[a] = npx - 1
        lo[tuple(sl0)] = first[tuple(sl0)]
        hi[tuple(sl1)] = last[tuple(sl1)]
        halos[(a, 0)] = lo.reshape((B,) + lo.shape[dim:])
        halos[(a, 1)] = hi.reshape((B,) + hi.shape[dim:])
    return halos


def fv_dt(P, pde, cfl, h, dim=3):
    """FV admissible dt: admissible_dt (kernels.py:267-281) with order 0 over
    patches, h = FV cell width (pinned reading of config 4)."""
    return batched.stable_dt_b(P, h, pde, 0, cfl, dim)


def fv_run(P0, pde, cells_per_axis, k, cfl, steps):
    P = P0.copy()
    h = 1.0 / cells_per_axis
    patch_edge = h * k
    log = {"dt": []}
    for _ in range(steps):
        dt = fv_dt(P, pde, cfl, h)
        P = batched.fv_update_b(P, pde, dt, (patch_edge,) * 3, fv_halos(P))
        log["dt"].append(dt)
    return P, log
