"""GPU coverage of every built (pde, dim, order) instantiation and the edge
cases of the operator API (empty batches, unconverged cells, NaN input)."""
import numpy as np
import pytest

from conftest import rel_linf

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def edg():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1806_07984_b200 as pkg
    return pkg


def _states(rng, name, dim, n, C):
    shape = (C,) + (n,) * dim
    if name == "euler":
        q = np.empty((C, dim + 2) + (n,) * dim)
        rho = 1.0 + 0.05 * rng.random(shape)
        q[:, 0] = rho
        for i in range(dim):
            q[:, 1 + i] = rho * (0.3 + 0.1 * i + 0.05 * rng.random(shape))
        q[:, 1 + dim] = 2.5 + 0.05 * rng.random(shape) + 0.5 * sum(q[:, 1 + i] ** 2 for i in range(dim)) / rho
        return q
    return (1.0 + 0.05 * rng.standard_normal(shape))[:, None]


# every order the reference accepts (basis.py:13-14: p in [1, 7]) in 2-D and 3-D
CASES = [(name, dim, p) for dim in (2, 3) for name in ("euler", "advection", "burgers") for p in range(1, 8)]


@pytest.mark.parametrize("name,dim,p", CASES)
def test_every_instantiation_matches_oracle(edg, name, dim, p):
    import torch
    from oracle import batched, ops
    rng = np.random.default_rng(100 * p + dim)
    C = 5
    Q = _states(rng, name, dim, p + 1, C)
    h = 1.0 / 27
    lam = 2.5 if name == "euler" else 1.2
    dt = 0.2 * h / ((2 * p + 1) * lam)
    opde = ops.make_pde(name, dim=dim) if name != "advection" else ops.advection((1.0, 0.5, 0.25)[:dim], dim)
    gpde = edg.pde.make_pde(name, dim=dim) if name != "advection" else edg.pde.advection((1.0, 0.5, 0.25)[:dim], dim)
    ref = batched.predictor_picard_b(Q, opde, dt, ops.basis_for(p), (h,) * dim)
    out = edg.kernels.stp_picard_batch(torch.from_numpy(Q).cuda(), gpde, dt, edg.basis.get_basis(p), (h,) * dim)
    torch.cuda.synchronize()
    assert np.array_equal(out["iterations"].cpu().numpy(), ref["iterations"])
    assert rel_linf(out["q_end"].cpu().numpy(), ref["q_end"]) < 1e-12
    keys = [(a, s) for a in range(dim) for s in (0, 1)]
    tf = out["trace_f"].cpu().numpy()
    for j, k in enumerate(keys):
        assert rel_linf(tf[:, j], ref["trace_f"][k]) < 1e-12


@pytest.mark.parametrize("dim,p,edges,C", [(2, 3, (1 / 27, 1 / 19), 7), (2, 3, (1 / 27, 1 / 27), 9),
                                           (3, 4, (1 / 16, 1 / 12, 1 / 20), 3), (2, 5, (1 / 27, 1 / 19), 4)])
def test_plane_predictors_anisotropic_ragged_mixed_convergence(edg, dim, p, edges, C):
    """The plane-task predictors (edg_stp2.cuh for 2-D n = 4, edg_stp3.cuh's
    plane tasks for 3-D n = 5) on anisotropic cells (1/h applied per axis
    inside the task instead of folded into the time coefficients), with a
    cell count that leaves the last CTA's work block ragged, and with cells
    of one block converging after different iteration counts (a smooth cell,
    a rough one): iteration counts equal the oracle's, values to 1e-12."""
    import torch
    from oracle import batched, ops
    rng = np.random.default_rng(7 * p + dim)
    Q = _states(rng, "euler", dim, p + 1, C)
    Q[0] = Q[0].mean(axis=tuple(range(1, dim + 1)), keepdims=True)      # constant cell: converges at once
    Q[-1, 0] *= 1.0 + 0.3 * rng.random(Q[-1, 0].shape)                    # rough cell: more iterations
    dt = 0.2 * min(edges) / ((2 * p + 1) * 2.5)
    ref = batched.predictor_picard_b(Q, ops.euler(dim), dt, ops.basis_for(p), edges)
    out = edg.kernels.stp_picard_batch(torch.from_numpy(Q).cuda(), edg.pde.euler(dim), dt, edg.basis.get_basis(p),
                                       edges)
    torch.cuda.synchronize()
    its = out["iterations"].cpu().numpy()
    assert np.array_equal(its, ref["iterations"])
    assert len(set(its.tolist())) > 1, "the cells were meant to converge at different iterations"
    assert np.array_equal(out["converged"].cpu().numpy().astype(bool), ref["converged"])
    assert rel_linf(out["q_end"].cpu().numpy(), ref["q_end"]) < 1e-12
    assert rel_linf(out["q_int"].cpu().numpy(), ref["q_int"]) < 1e-12
    keys = [(a, s) for a in range(dim) for s in (0, 1)]
    tq, tf = out["trace_q"].cpu().numpy(), out["trace_f"].cpu().numpy()
    for j, k in enumerate(keys):
        assert rel_linf(tq[:, j], ref["trace_q"][k]) < 1e-12
        assert rel_linf(tf[:, j], ref["trace_f"][k]) < 1e-12


@pytest.mark.parametrize("p", [6, 7])
def test_3d_high_order_steps_vs_oracle(edg, p):
    """3-D Euler at the paper's highest orders (Table 1 measures p = 7,
    PAPER.md:1788-1793): two whole steps on a 3^3 outflow grid against the
    oracle's Algorithm-1 driver."""
    from oracle import drivers, ops
    cfg = edg.configs.CONFIGS["cfg3"].with_(cells=3, order=p)
    Q0 = edg.configs.initial_dg_uniform(cfg)
    s = edg.solver.DGSolver(edg.pde.euler(3), p, edg.mesh.CartesianMesh(3, 3, False), cfg.cfl)
    s.set_state(Q0)
    s.run(2, graph=False)
    s.check_status()
    Qo, log = drivers.dg_uniform_run(Q0, ops.euler(3), p, 3, 3, False, cfg.cfl, 2)
    assert rel_linf(s.state().cpu().numpy(), Qo) <= 1e-10
    assert rel_linf(s.dt_history(), np.array(log["dt"])) <= 1e-13
    assert np.array_equal(s.iterations.cpu().numpy(), log["iterations"][-1])


def test_empty_batches(edg):
    import torch
    b = edg.basis.get_basis(3)
    pde = edg.pde.euler(2)
    out = edg.kernels.stp_picard_batch(torch.empty((0, 4, 4, 4), dtype=torch.float64, device="cuda"), pde, 1e-3, b,
                                       (0.1, 0.1))
    assert out["q_end"].shape[0] == 0
    r = edg.kernels.riemann_rusanov_batch(torch.empty((0, 4, 4), dtype=torch.float64, device="cuda"),
                                          torch.empty((0, 4, 4), dtype=torch.float64, device="cuda"), pde, 0)
    assert r.shape[0] == 0


def test_unconverged_cells_flagged_like_reference(edg, golden_ops):
    """Cases 5-7 of the golden vectors hit max_iter without converging
    (kernels.py:158-159): converged=False, iterations=max_iter."""
    import torch
    for ci in (5, 6, 7):
        g = lambda k: golden_ops[f"stp{ci}_{k}"]  # noqa: E731
        dim, p, code = (int(v) for v in g("meta"))
        name = {0: "advection", 1: "burgers", 2: "euler"}[code]
        pde = edg.pde.make_pde(name, dim=dim) if name != "advection" else edg.pde.advection((1.0, 0.5, 0.25)[:dim], dim)
        out = edg.kernels.stp_picard_batch(torch.from_numpy(g("q")).cuda(), pde, float(g("dt")),
                                           edg.basis.get_basis(p), tuple(g("edges")))
        assert not out["converged"].any()
        assert np.array_equal(out["iterations"].cpu().numpy(), g("iterations"))


def test_nan_input_propagates_and_is_counted(edg):
    """The reference lets NaN propagate silently; the GPU solver does the same
    and counts non-finite cells (NumericalError on check_status)."""
    cfg = edg.configs.CONFIGS["cfg2"].with_(cells=9)
    Q0 = edg.configs.initial_dg_uniform(cfg)
    Q0[40, 0, 2, 2] = np.nan
    s = edg.solver.DGSolver(edg.pde.euler(2), cfg.order, edg.mesh.CartesianMesh(9, 2, True), 0.2)
    s.set_state(Q0)
    s.run(2, graph=False)
    it = s.iterations.cpu().numpy()
    assert it[40] == 2 * (cfg.order + 1)          # NaN delta never converges (kernels.py:143-147)
    with pytest.raises(edg.errors.NumericalError):
        s.check_status()
    assert np.isnan(s.state().cpu().numpy()[40]).any()


@pytest.mark.slow
def test_cfg5_full_mesh_two_steps_vs_oracle(edg):
    from oracle import drivers, ops, spacetree
    cfg = edg.configs.CONFIGS["cfg5"]
    cells = edg.configs.amr_cells(cfg)
    mesh = edg.mesh.AdaptiveMesh(cells, 2, True)
    s = edg.solver.DGSolver(edg.pde.euler(2), cfg.order, mesh, cfg.cfl)
    Q0 = edg.configs.initial_dg_amr(cfg, mesh.cells)
    s.set_state(Q0)
    s.run(2, graph=True)
    s.check_status()
    forest = spacetree.FaceForest(cells, 2, True)
    Qo, log = drivers.dg_amr_run(forest, {k: Q0[i] for i, k in enumerate(forest.sfc)}, ops.euler(2), cfg.order,
                                 cfg.cfl, 2)
    assert rel_linf(s.state().cpu().numpy(), np.stack([Qo[k] for k in forest.sfc])) <= 1e-10
