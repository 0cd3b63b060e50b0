"""GPU parity of the cell-local dynamic-AMR operators (SURVEY.md section 8(f)
f2; transfer.py:99-158) through the C ABI against the reference's own
outputs (tests/golden/amr.npz) and the oracle."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "amr.npz"))
CASES = range(int(G["amr_ncases"]))
TOL = 1e-13   # fp64 contraction order differs from numpy's tensordot (BLAS)


@pytest.fixture(scope="module")
def tr():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_1806_07984_b200 import _lib, transfer
    _lib.load()
    return transfer


def _rel(a, b):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b))) / max(1e-300, np.max(np.abs(b))))


@pytest.mark.parametrize("ci", CASES)
def test_indicator_and_verdicts_vs_reference(tr, ci):
    dim, p, m, C = (int(v) for v in G[f"amr{ci}_meta"])
    Q = G[f"amr{ci}_q"]
    rt, ct, ml, mnl = G["amr_decision"]
    dec = tr.RefinementDecision(refine_tol=rt, coarsen_tol=ct, max_level=int(ml))
    ind, ver = tr.gradient_indicator_batch(Q, p, G[f"amr{ci}_levels"], dec, int(mnl))
    ind = ind.cpu().numpy()
    ref = G[f"amr{ci}_ind"]
    assert np.all(np.abs(ind - ref) <= TOL * np.maximum(1.0, np.abs(ref)))
    assert np.array_equal(ver.cpu().numpy(), G[f"amr{ci}_verdict"])
    # single-cell API (reference signatures)
    assert abs(tr.gradient_indicator(Q[0], p) - ref[0]) <= TOL * max(1.0, abs(ref[0]))
    code = {1: tr.RefinementDecision.REFINE, 0: tr.RefinementDecision.KEEP, -1: tr.RefinementDecision.COARSEN}
    for c in range(C):
        v = tr.evaluate_refinement_criterion(Q[c], int(G[f"amr{ci}_levels"][c]), p, dec, int(mnl))
        assert v == code[int(G[f"amr{ci}_verdict"][c])]


@pytest.mark.parametrize("ci", CASES)
def test_interpolate_and_restrict_volume_vs_reference(tr, ci):
    dim, p, m, C = (int(v) for v in G[f"amr{ci}_meta"])
    ops = tr.get_transfer(p)
    digits = list(np.ndindex(*(3,) * dim))
    Q = G[f"amr{ci}_q"]
    # batched: all 3^d children of parent 0
    out = tr.interpolate_volume_batch(p, Q, digits, parent=[0] * len(digits)).cpu().numpy()
    assert _rel(out, G[f"amr{ci}_interp"]) <= TOL
    # single child through the reference signature
    assert _rel(tr.interpolate_volume(ops, Q[0], digits[-1]), G[f"amr{ci}_interp"][-1]) <= TOL
    ch = G[f"amr{ci}_children"]
    r = tr.restrict_volume_batch(p, ch[None]).cpu().numpy()[0]
    assert _rel(r, G[f"amr{ci}_restrict"]) <= TOL
    children = {dg: ch[i] for i, dg in enumerate(digits)}
    assert _rel(tr.restrict_volume(ops, children), G[f"amr{ci}_restrict"]) <= TOL
    # another dict order sums in that order (same value to rounding)
    rev = dict(reversed(list(children.items())))
    assert _rel(tr.restrict_volume(ops, rev), G[f"amr{ci}_restrict"]) <= 1e-12


@pytest.mark.parametrize("ci", CASES)
def test_refine_coarsen_round_trip_on_device(tr, ci):
    dim, p, m, C = (int(v) for v in G[f"amr{ci}_meta"])
    Q = G[f"amr{ci}_q"]
    digits = list(np.ndindex(*(3,) * dim))
    kids = tr.interpolate_volume_batch(p, Q, digits * C, parent=np.repeat(np.arange(C), len(digits)))
    back = tr.restrict_volume_batch(p, kids.reshape((C, len(digits)) + Q.shape[1:])).cpu().numpy()
    assert np.max(np.abs(back - Q)) <= 1e-12 * max(1.0, np.max(np.abs(Q)))


def test_indicator_nan_axis_dropped_and_errors(tr):
    import torch
    from paper_1806_07984_b200.errors import ConfigError
    from oracle import transfer as ot
    rng = np.random.default_rng(5)
    q = rng.standard_normal((4, 5, 5))
    q[0, 2, 3] = np.nan      # NaN in every axis through node (2, 3)
    ref = ot.gradient_indicator(q, 4)
    got = tr.gradient_indicator(q, 4)
    assert (np.isnan(ref) and np.isnan(got)) or got == ref
    with pytest.raises(ValueError):
        tr.RefinementDecision(refine_tol=0.1, coarsen_tol=0.2, max_level=3)
    with pytest.raises(ConfigError):
        tr.gradient_indicator_batch(torch.zeros((1, 1, 10, 10), dtype=torch.float64, device="cuda"), 9)
    empty = tr.gradient_indicator_batch(torch.zeros((0, 4, 4, 4), dtype=torch.float64, device="cuda"), 3)
    assert empty.numel() == 0


def _keys(a):
    return [(int(r[0]), (int(r[1]), int(r[2]))) for r in a]


@pytest.mark.parametrize("mi", range(int(G["mesh_ncases"])))
def test_apply_mesh_updates_vs_reference(tr, mi):
    """transfer.py:195-219 on the reference's mesh and verdicts: same new
    cells, new data within 1e-13, solutions dict updated like the reference."""
    from paper_1806_07984_b200 import amr
    from paper_1806_07984_b200.mesh import AdaptiveMesh
    pre = f"mesh{mi}_"
    p = int(G[pre + "order"])
    cells0 = _keys(G[pre + "cells0"])
    mesh = AdaptiveMesh(cells0, 2, True)
    code = {1: amr.REFINE, 0: amr.KEEP, -1: amr.COARSEN}
    verdicts = {k: code[int(v)] for k, v in zip(_keys(G[pre + "verdict_keys"]), G[pre + "verdicts"])}
    sol = {k: G[pre + "sol0"][i] for i, k in enumerate(cells0)}
    delta, new = amr.apply_mesh_updates(mesh, verdicts, sol, p)
    assert sorted(new) == _keys(G[pre + "new_keys"])
    ref = G[pre + "new_data"]
    got = np.stack([new[k] for k in sorted(new)])
    assert _rel(got, ref) <= TOL
    assert sorted(sol) == _keys(G[pre + "cells1"])
    assert sorted(delta.created_cells) == _keys(G[pre + "created"])


def test_solver_adapt_moves_state_and_steps(tr):
    """amr.adapt: verdicts on the device, kept cells bit-identical, refined /
    coarsened cells equal to the batch operators, and the new solver steps
    (checked against the oracle driver on the adapted mesh for one step)."""
    import torch
    from paper_1806_07984_b200 import amr, configs, mesh as M, pde, solver
    cfg = configs.CONFIGS["cfg5"].with_(cells=27)
    mesh = M.AdaptiveMesh(configs.amr_cells(cfg), 2, True)
    s = solver.DGSolver(pde.euler(2), cfg.order, mesh, cfg.cfl)
    Q0 = configs.initial_dg_amr(cfg, mesh.cells)
    s.set_state(Q0)
    s.step()
    s.check_status()
    Q1 = s.state().clone()
    # thresholds from the indicators: refine the roughest base cells, let
    # smooth fine clusters merge back (min_level 3 keeps the base level, so no
    # face gets two levels between its sides)
    ind = tr.gradient_indicator_batch(Q1, cfg.order).cpu().numpy()
    lv = mesh.levels
    rt = float(np.quantile(ind[lv == lv.min()], 0.9))
    ct = min(float(np.quantile(ind[lv == lv.max()], 0.6)), 0.5 * rt)
    dec = tr.RefinementDecision(refine_tol=rt, coarsen_tol=ct, max_level=int(lv.max()))
    new, delta = amr.adapt(s, dec, min_level=int(lv.min()), in_place=False)
    assert new.mesh is not s.mesh and s.mesh.ncells == mesh.ncells
    assert delta.created_cells and delta.removed_cells
    assert new.mesh.ncells == mesh.ncells - len(delta.removed_cells) + len(delta.created_cells)
    Qn = new.state()
    for key in new.mesh.cells:
        if key in mesh.pos:
            assert torch.equal(Qn[new.mesh.pos[key]], Q1[mesh.pos[key]])
    refined = [c for c in delta.removed_cells if all(k in new.mesh.pos for k in new.mesh.child_keys(c))]
    merged = [c for c in delta.created_cells if c in new.mesh.pos and c not in mesh.pos
              and all(k in mesh.pos for k in mesh.child_keys(c))]
    assert refined
    for c in refined[:3]:
        want = tr.interpolate_volume_batch(cfg.order, Q1[[mesh.pos[c]]], list(np.ndindex(3, 3)), [0] * 9)
        got = torch.stack([Qn[new.mesh.pos[k]] for k in new.mesh.child_keys(c)])
        assert torch.equal(got, want)
    for c in merged[:3]:
        want = tr.restrict_volume_batch(cfg.order, Q1[[mesh.pos[k] for k in mesh.child_keys(c)]][None])[0]
        assert torch.equal(Qn[new.mesh.pos[c]], want)
    new.step()
    new.check_status()
    assert torch.isfinite(new.state()).all()


def test_solver_adapt_in_place_reuses_the_solver(tr):
    """amr.adapt(in_place=True): the same DGSolver adopts the adapted mesh
    (DGSolver.remesh), its state equals the rebuilt-solver path bitwise, and
    both step to identical bits."""
    import torch
    from paper_1806_07984_b200 import amr, configs, mesh as M, pde, solver
    cfg = configs.CONFIGS["cfg5"].with_(cells=27)
    mesh = M.AdaptiveMesh(configs.amr_cells(cfg), 2, True)
    Q0 = configs.initial_dg_amr(cfg, mesh.cells)
    a = solver.DGSolver(pde.euler(2), cfg.order, mesh, cfg.cfl)
    b = solver.DGSolver(pde.euler(2), cfg.order, mesh, cfg.cfl)
    for s in (a, b):
        s.set_state(Q0)
        s.run(2, graph=True)
    ind = tr.gradient_indicator_batch(a.state(), cfg.order).cpu().numpy()
    lv = mesh.levels
    dec = tr.RefinementDecision(refine_tol=float(np.quantile(ind[lv == lv.min()], 0.9)),
                                coarsen_tol=0.0, max_level=int(lv.max()) + 1)
    new_b, _ = amr.adapt(b, dec, min_level=int(lv.min()), in_place=False)
    same, delta = amr.adapt(a, dec, min_level=int(lv.min()))
    assert same is a and a.mesh.ncells == new_b.mesh.ncells and delta.created_cells
    assert a.mesh.max_chain >= 1
    assert torch.equal(a.state(), new_b.state())
    for s in (a, new_b):
        s.run(2, graph=True)
        s.check_status()
    torch.cuda.synchronize()
    assert torch.equal(a.state(), new_b.state())


@pytest.mark.parametrize("name", ["deep2d", "deep3d"])
def test_deep_chain_steps_vs_oracle(name):
    """Multi-level hanging-face chains (mesh.py:67-100) on the device: three
    steps on the reference's two-level-jump meshes (tests/golden/mesh_deep.json)
    against the oracle's level-by-level interpolation / restriction, and the
    periodic 2-D run conserves every component's integral."""
    import json
    import os
    import torch
    from oracle import drivers, ops, spacetree
    from paper_1806_07984_b200 import mesh as M, pde, solver
    ref = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "mesh_deep.json")))[name]
    cells = [(l, tuple(ix)) for l, ix in ref["sfc"]]
    dim, p = ref["dim"], 3
    mesh = M.AdaptiveMesh(cells, dim, ref["periodic"])
    assert mesh.max_chain == 2
    rng = np.random.default_rng(11)
    Q0 = np.empty((mesh.ncells, dim + 2) + (p + 1,) * dim)
    Q0[:, 0] = 1.0 + 0.1 * rng.random(Q0[:, 0].shape)
    for i in range(dim):
        Q0[:, 1 + i] = Q0[:, 0] * (0.3 + 0.1 * rng.random(Q0[:, 0].shape))
    Q0[:, 1 + dim] = 2.5 + 0.5 * sum(Q0[:, 1 + i] ** 2 for i in range(dim)) / Q0[:, 0]
    s = solver.DGSolver(pde.euler(dim), p, mesh, 0.2)
    s.set_state(Q0)
    s.run(3, graph=False)
    s.check_status()
    torch.cuda.synchronize()
    forest = spacetree.FaceForest(cells, dim, ref["periodic"])
    Qo, log = drivers.dg_amr_run(forest, {k: Q0[i] for i, k in enumerate(forest.sfc)}, ops.euler(dim), p, 0.2, 3)
    Qo = np.stack([Qo[k] for k in forest.sfc])
    G = s.state().cpu().numpy()
    assert np.abs(G - Qo).max() / np.abs(Qo).max() <= 1e-10
    assert np.abs(s.dt_history() - np.array(log["dt"])).max() <= 1e-13 * max(log["dt"])
    if ref["periodic"]:
        b = ops.basis_for(p)
        w = np.multiply.outer(b.weights, b.weights)
        vol = (3.0 ** -mesh.levels.astype(float)) ** dim
        mass = lambda Q: ((Q * w).sum(axis=(2, 3)) * vol[:, None]).sum(axis=0)  # noqa: E731
        assert np.allclose(mass(G), mass(Q0), rtol=1e-13, atol=1e-15)
