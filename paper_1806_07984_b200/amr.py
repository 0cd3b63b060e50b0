"""Dynamic AMR on the GPU -- mirror of the reference's mesh-update path
(/root/reference/pkg/src/enclavedg/transfer.py:161-219, SURVEY.md section
8(f) f2) on AdaptiveMesh.

The refine / keep / coarsen verdicts come from the device kernel behind
transfer.gradient_indicator_batch (edg_gradient_indicator), the volumetric
data move with edg_interpolate_volume / edg_restrict_volume; only the
topology bookkeeping (which cells split or merge) is host work, as in the
reference.  Differences from the reference API: cells are addressed by their
(level, index) keys instead of spacetree node objects, and hanging-face
chains may span up to mesh.MAX_CHAIN levels (ConfigError beyond).
"""
from __future__ import annotations

import logging

import numpy as np

from . import transfer as T
from .kernels import _dev, _torch
from .mesh import AdaptiveMesh

log = logging.getLogger(__name__)
REFINE, KEEP, COARSEN = T.RefinementDecision.REFINE, T.RefinementDecision.KEEP, T.RefinementDecision.COARSEN
_CODE = {1: REFINE, 0: KEEP, -1: COARSEN}


def plan_mesh_updates(mesh: AdaptiveMesh, verdicts: dict):
    """transfer.py:161-192: refine keys in verdict order; a parent is
    coarsened only if all 3^d children are real cells voting COARSEN (a
    refined child or a dissenting vote skips the cluster, logged)."""
    refine, coarsen, seen = [], [], set()
    nchild = 3 ** mesh.dim
    for key, verdict in verdicts.items():
        if key not in mesh.pos:
            continue
        if verdict == REFINE:
            refine.append(key)
        elif verdict == COARSEN:
            parent = mesh.parent_key(key)
            if parent is None or parent in seen:
                continue
            seen.add(parent)
            kids = mesh.child_keys(parent)
            real = [k for k in kids if k in mesh.pos]
            if len(real) != nchild:
                log.info("coarsening of %r skipped: refined sibling present", parent)
                continue
            votes = [verdicts.get(k) == COARSEN for k in kids]
            if all(votes):
                coarsen.append(parent)
            else:
                log.info("coarsening of %r skipped: %d of %d siblings agree", parent, sum(votes), len(votes))
    return refine, coarsen


def apply_mesh_updates(mesh: AdaptiveMesh, verdicts: dict, solutions: dict, order: int):
    """transfer.py:195-219: apply the verdicts, moving the volumetric data with
    the topology.  solutions maps cell key -> (m, n^d) array (numpy or CUDA
    tensor); dropped keys are removed from it and the new cells' data added.
    Returns (MeshDelta, new_data)."""
    torch = _torch()
    refine, coarsen = plan_mesh_updates(mesh, verdicts)
    new_data = {}
    if refine:
        Q = torch.stack([_dev(solutions[k])[0] for k in refine])
        digits = list(np.ndindex(*(3,) * mesh.dim))
        kids = T.interpolate_volume_batch(order, Q, digits * len(refine),
                                          parent=np.repeat(np.arange(len(refine)), len(digits)))
        i = 0
        for k in refine:
            for ck in mesh.child_keys(k):
                new_data[ck] = kids[i]
                i += 1
    if coarsen:
        ch = torch.stack([torch.stack([_dev(solutions[ck])[0] for ck in mesh.child_keys(p)]) for p in coarsen])
        par = T.restrict_volume_batch(order, ch)
        for i, p in enumerate(coarsen):
            new_data[p] = par[i]
    host = bool(solutions) and isinstance(next(iter(solutions.values())), np.ndarray)
    if host:
        new_data = {k: v.cpu().numpy() for k, v in new_data.items()}
    delta = mesh.update_topology(refine, coarsen)
    for key in delta.removed_cells:
        solutions.pop(key, None)
    solutions.update(new_data)
    return delta, new_data


def adapt(solver, decision: T.RefinementDecision, min_level: int = 0, in_place: bool = True, **solver_kw):
    """One adaptation of a device-resident DGSolver on an AdaptiveMesh:
    indicator and verdicts of every cell on the GPU, the plan on the host,
    the new state assembled on the GPU (kept cells gathered, refined cells
    interpolated, coarsened clusters restricted).  With in_place (default)
    the solver itself adopts the updated mesh (DGSolver.remesh: device tables
    rebuilt, buffers reused while they fit); otherwise a new solver is built
    and the old one keeps its mesh.  Returns (solver, MeshDelta)."""
    import copy

    from .solver import DGSolver
    torch = _torch()
    if not isinstance(solver.mesh, AdaptiveMesh):
        raise TypeError("adapt needs a DGSolver on an AdaptiveMesh")
    mesh = copy.copy(solver.mesh)   # the old solver keeps its own, unchanged mesh
    old_cells, old_pos = list(mesh.cells), dict(mesh.pos)
    Q = solver.state()
    _, v = T.gradient_indicator_batch(Q, solver.order, mesh.levels, decision, min_level)
    v = v.cpu().numpy()
    verdicts = {key: _CODE[int(v[i])] for i, key in enumerate(old_cells)}
    refine, coarsen = plan_mesh_updates(mesh, verdicts)
    kids = par = None
    if refine:
        ridx = torch.tensor([old_pos[k] for k in refine], dtype=torch.int32, device="cuda")
        digits = list(np.ndindex(*(3,) * mesh.dim))
        kids = T.interpolate_volume_batch(solver.order, Q, digits * len(refine),
                                          parent=ridx.cpu().numpy().repeat(len(digits)))
    if coarsen:
        cidx = torch.tensor([[old_pos[ck] for ck in mesh.child_keys(p)] for p in coarsen], dtype=torch.long,
                            device="cuda")
        par = T.restrict_volume_batch(solver.order, Q[cidx])
    delta = mesh.update_topology(refine, coarsen)
    newQ = torch.empty((mesh.ncells,) + tuple(Q.shape[1:]), dtype=torch.float64, device="cuda")
    kept = [k for k in mesh.cells if k in old_pos]
    if kept:
        dst = torch.tensor([mesh.pos[k] for k in kept], dtype=torch.long, device="cuda")
        src = torch.tensor([old_pos[k] for k in kept], dtype=torch.long, device="cuda")
        newQ[dst] = Q[src]
    if refine:
        dst = torch.tensor([mesh.pos[ck] for k in refine for ck in mesh.child_keys(k)], dtype=torch.long,
                           device="cuda")
        newQ[dst] = kids
    if coarsen:
        dst = torch.tensor([mesh.pos[p] for p in coarsen], dtype=torch.long, device="cuda")
        newQ[dst] = par
    if in_place:
        solver.remesh(mesh, newQ)
        return solver, delta
    kw = dict(tol=solver.tol, max_iter=solver.max_iter or None, check_finite=solver.check_finite,
              max_steps=solver.max_steps, two_streams=getattr(solver, "two_streams", True))
    kw.update(solver_kw)
    new = DGSolver(solver.pde, solver.order, mesh, solver.cfl, **kw)
    new.set_state(newQ)
    return new, delta
