"""Pin the CPU oracle against vectors produced by the reference package
(tests/golden/make_golden.py).  CPU only."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, rel_linf
from oracle import ops, batched, drivers, transfer, spacetree
from paper_1806_07984_b200 import configs as cf

PDES = {0: "advection", 1: "burgers", 2: "euler"}


def _pde(code, dim):
    if PDES[code] == "advection":
        return ops.advection(velocity=(1.0, 0.5, 0.25)[:dim], dim=dim)
    return ops.make_pde(PDES[code], dim=dim)


def test_basis_and_time_operators_bitwise(golden_ops):
    for p in range(1, 8):
        b = ops.basis_for(p)
        assert np.array_equal(b.nodes, golden_ops[f"basis{p}_nodes"])
        assert np.array_equal(b.weights, golden_ops[f"basis{p}_weights"])
        assert np.array_equal(b.diff_matrix, golden_ops[f"basis{p}_D"])
        assert np.array_equal(b.trace_left, golden_ops[f"basis{p}_tl"])
        assert np.array_equal(b.trace_right, golden_ops[f"basis{p}_tr"])
        kinv, lift = ops.time_operators(b)
        assert np.array_equal(kinv, golden_ops[f"basis{p}_kinv"])
        assert np.array_equal(lift, golden_ops[f"basis{p}_lift"])
        t = transfer.transfer_for(p)
        assert np.array_equal(np.stack(t.interp), golden_ops[f"basis{p}_interp"])
        assert np.array_equal(np.stack(t.restrict), golden_ops[f"basis{p}_restrict"])


def test_spec_gauss_legendre_examples():
    # SPEC.md:233-236
    x, w = ops.gl_rule(2)
    assert np.allclose(x, [0.5 - 1 / (2 * np.sqrt(3)), 0.5 + 1 / (2 * np.sqrt(3))], atol=1e-15)
    assert np.allclose(w, [0.5, 0.5], atol=1e-16)
    x, w = ops.gl_rule(3)
    assert abs((w * x ** 5).sum() - 1 / 6) < 1e-15
    with pytest.raises(ops.OracleConfigError):
        ops.gl_rule(17)
    with pytest.raises(ops.OracleConfigError):
        ops.Basis(8)


def _trace_keys(dim):
    return [(a, s) for a in range(dim) for s in (0, 1)]


@pytest.mark.parametrize("ci", range(8))
def test_stp_picard_percell_bitwise(golden_ops, ci):
    g = lambda k: golden_ops[f"stp{ci}_{k}"]  # noqa: E731
    dim, p, code = (int(v) for v in g("meta"))
    pde = _pde(code, dim)
    b = ops.basis_for(p)
    Q, dt, edges = g("q"), float(g("dt")), tuple(g("edges"))
    for c in range(Q.shape[0]):
        st = ops.predictor_picard(Q[c], pde, dt, b, edges)
        assert st.iterations == g("iterations")[c]
        assert st.converged == bool(g("converged")[c])
        assert np.array_equal(st.q_end, g("q_end")[c])
        assert np.array_equal(st.q_int, g("q_int")[c])
        for j, key in enumerate(_trace_keys(dim)):
            assert np.array_equal(st.trace_q[key], g("trace_q")[c, j])
            assert np.array_equal(st.trace_f[key], g("trace_f")[c, j])
        outc = {key: g("outcomes")[c, j] for j, key in enumerate(_trace_keys(dim))}
        assert np.array_equal(ops.correct(st, outc, b, edges), g("corrected")[c])
        with pytest.raises(AssertionError):
            ops.correct(st, {}, b, edges)
    if pde.is_linear:
        for c in range(Q.shape[0]):
            ck = ops.predictor_ck(Q[c], pde, dt, b, edges)
            assert np.array_equal(ck.q_end, g("ck_q_end")[c])


@pytest.mark.parametrize("ci", range(8))
def test_stp_picard_batched_matches(golden_ops, ci):
    g = lambda k: golden_ops[f"stp{ci}_{k}"]  # noqa: E731
    dim, p, code = (int(v) for v in g("meta"))
    pde = _pde(code, dim)
    b = ops.basis_for(p)
    out = batched.predictor_picard_b(g("q"), pde, float(g("dt")), b, tuple(g("edges")))
    assert np.array_equal(out["iterations"], g("iterations"))
    assert rel_linf(out["q_end"], g("q_end")) <= 1e-14
    for j, key in enumerate(_trace_keys(dim)):
        assert rel_linf(out["trace_f"][key], g("trace_f")[:, j]) <= 1e-14
        assert rel_linf(out["trace_q"][key], g("trace_q")[:, j]) <= 1e-14


def test_picard_equals_ck_for_linear(golden_ops):
    # Picard with tol -> 0 reproduces CK on a linear PDE
    g = lambda k: golden_ops[f"stp0_{k}"]  # noqa: E731
    pde = ops.advection()
    b = ops.basis_for(3)
    for c in range(3):
        st = ops.predictor_picard(g("q")[c], pde, float(g("dt")), b, tuple(g("edges")), tol=1e-15, max_iter=60)
        assert rel_linf(st.q_end, g("ck_q_end")[c]) < 1e-12


def test_riemann_bitwise(golden_ops):
    for ci, code, dim, axis in golden_ops["riem_index"]:
        key = f"riem{ci}_{axis}_"
        pde = _pde(int(code), int(dim))
        lo, hi = golden_ops[key + "lo"], golden_ops[key + "hi"]
        for c in range(lo.shape[0]):
            o = ops.rusanov(lo[c], hi[c], pde, int(axis))
            assert np.array_equal(o, golden_ops[key + "out"][c])
            assert np.array_equal(ops.rusanov(lo[c], hi[c], pde, int(axis), sign=-1), golden_ops[key + "neg"][c])
            assert np.array_equal(-o, golden_ops[key + "neg"][c])


def test_spec_rusanov_and_dt_examples(golden_ops):
    adv = ops.advection()
    assert np.array_equal(ops.rusanov(np.full((1, 4), 2.0), np.full((1, 4), 2.0), adv, 0),
                          golden_ops["kat_rusanov_adv_equal"])
    assert np.all(golden_ops["kat_rusanov_adv_equal"] == 2.0)
    assert np.all(golden_ops["kat_rusanov_adv_upwind"] == 1.0)
    assert np.all(golden_ops["kat_rusanov_burgers"] == 3.0)
    assert np.array_equal(ops.rusanov(np.full((1, 4), 2.0), np.full((1, 4), 0.0), ops.burgers(), 0),
                          golden_ops["kat_rusanov_burgers"])
    # SPEC.md:306
    dt = ops.stable_dt(((1 / 9, np.ones((1, 4, 4))) for _ in range(81)), ops.advection((1.0, 0.0)), 3, 0.9, 2)
    assert dt == float(golden_ops["kat_dt_adv_h9"])
    assert abs(dt - 0.9 / 63) < 1e-16


def test_admissible_dt_nan_and_zero_speed(golden_ops):
    pde = ops.euler(2)
    Q = golden_ops["dt_euler_q"]
    dt = ops.stable_dt(((1 / 9, Q[c]) for c in range(Q.shape[0])), pde, 3, 0.9, 2)
    assert dt == float(golden_ops["dt_euler_val"])
    assert batched.stable_dt_b(Q, 1 / 9, pde, 3, 0.9, 2) == dt
    with pytest.raises(ops.OracleNoWaveSpeed):
        ops.stable_dt(((1 / 9, np.zeros((4, 4, 4)) + [[[1.0]], [[0.0]], [[0.0]], [[0.0]]]),), pde, 3, 0.9, 2)


@pytest.mark.parametrize("ci", range(3))
def test_fv_patch_bitwise(golden_ops, ci):
    key = f"fv{ci}_"
    dim, k, code = (int(v) for v in golden_ops[key + "meta"])
    pde = _pde(code, dim)
    P, H = golden_ops[key + "patch"], golden_ops[key + "halos"]
    dt = float(golden_ops[key + "dt"])
    for c in range(P.shape[0]):
        halos = {kk: H[c, j] for j, kk in enumerate(_trace_keys(dim))}
        assert np.array_equal(ops.fv_update(P[c], pde, dt, (1 / 16,) * dim, halos), golden_ops[key + "out"][c])
        lay = ops.boundary_layers(P[c])
        for j, kk in enumerate(_trace_keys(dim)):
            assert np.array_equal(lay[kk], golden_ops[key + "layers"][c, j])
    halos = {kk: H[:, j] for j, kk in enumerate(_trace_keys(dim))}
    assert np.array_equal(batched.fv_update_b(P, pde, dt, (1 / 16,) * dim, halos), golden_ops[key + "out"])
    with pytest.raises(ops.OracleNotReady):
        ops.fv_update(P[0], pde, dt, (1 / 16,) * dim, {})


def test_transfer_functions_bitwise(golden_ops):
    for p in (2, 3, 4):
        t = transfer.transfer_for(p)
        tr2, tr3 = golden_ops[f"xfer{p}_tr2"], golden_ops[f"xfer{p}_tr3"]
        for j in range(3):
            assert np.array_equal(transfer.interp_trace(t, tr2, (j,)), golden_ops[f"xfer{p}_i2_{j}"])
            assert np.array_equal(transfer.restrict_trace(t, tr2, (j,)), golden_ops[f"xfer{p}_r2_{j}"])
            for l in range(3):
                assert np.array_equal(transfer.interp_trace(t, tr3, (j, l)), golden_ops[f"xfer{p}_i3_{j}{l}"])
                assert np.array_equal(transfer.restrict_trace(t, tr3, (j, l)), golden_ops[f"xfer{p}_r3_{j}{l}"])
        buf = transfer.ParentAccumulator()
        for j in range(3):
            transfer.accumulate_restriction(t, buf, tr2 * (j + 1), (j,), 7)
        assert np.array_equal(buf.outcome, golden_ops[f"xfer{p}_acc2"])
        with pytest.raises(AssertionError):
            transfer.accumulate_restriction(t, buf, tr2, (0,), 7)


def test_transfer_adjointness():
    # SPEC.md:191 / 594: <interp u, v>_children = <u, restrict v>_parent
    rng = np.random.default_rng(3)
    for p in range(1, 6):
        t = transfer.transfer_for(p)
        w = t.basis.weights
        u = rng.standard_normal(p + 1)
        lhs = rhs = 0.0
        for j in range(3):
            v = rng.standard_normal(p + 1)
            lhs += (w / 3.0 * (t.interp[j] @ u) * v).sum()
            rhs += (w * u * (t.restrict[j] @ v)).sum()
        assert abs(lhs - rhs) < 1e-12


def test_cfg1_full_trajectory_matches_reference(golden_traj):
    cfg = cf.CONFIGS["cfg1"]
    Q0 = cf.initial_dg_uniform(cfg)
    assert np.array_equal(Q0, golden_traj["cfg1_q0"])
    Q, log = drivers.dg_uniform_run(Q0, ops.advection(cfg.velocity), cfg.order, cfg.cells, 2, True,
                                    cfg.cfl, cfg.steps)
    assert np.array_equal(np.array(log["dt"]), golden_traj["cfg1_dt"])
    assert rel_linf(Q, golden_traj["cfg1_q"]) < 1e-13


@pytest.mark.parametrize("tag", ["cfg2p", "cfg2s", "cfg3w"])
def test_dg_proxy_trajectories(golden_traj, tag):
    N, dim, p, periodic, steps, cells, wlo = (int(v) for v in golden_traj[tag + "_meta"])
    cfl = float(golden_traj[tag + "_cfl"])
    base = {"cfg2p": "cfg2", "cfg2s": "cfg2", "cfg3w": "cfg3"}[tag]
    cfg = cf.CONFIGS[base].with_(cells=cells, cfl=cfl)
    Q0 = cf.initial_dg_uniform(cfg, window=None if wlo < 0 else (wlo, N))
    assert np.array_equal(Q0, golden_traj[tag + "_q0"])
    h = 1.0 / cells
    Q, log = drivers.dg_uniform_run(Q0, ops.euler(dim), p, N, dim, bool(periodic), cfl, steps, h=h)
    assert np.array_equal(np.stack(log["iterations"]), golden_traj[tag + "_its"])
    assert rel_linf(np.array(log["dt"]), golden_traj[tag + "_dt"]) < 1e-14
    assert rel_linf(Q, golden_traj[tag + "_q"]) < 1e-13
    # the per-cell structure (used by the CPU baseline) agrees too
    b = ops.basis_for(p)
    Qp, dtp, _ = drivers.dg_uniform_step_percell(Q0, ops.euler(dim), b, N, dim, bool(periodic), cfl, h=h)
    Qb, dtb, _ = drivers.dg_uniform_step(Q0, ops.euler(dim), b, N, dim, bool(periodic), cfl, h=h)
    assert dtp == dtb and rel_linf(Qp, Qb) < 1e-14


def test_fv_proxy_trajectory_bitwise(golden_traj):
    cfg = cf.CONFIGS["cfg4"].with_(cells=16)
    P0 = cf.initial_fv(cfg)
    assert np.array_equal(P0, golden_traj["cfg4p_q0"])
    P, log = drivers.fv_run(P0, ops.euler(3), 16, 8, cfg.cfl, 5)
    assert np.array_equal(np.array(log["dt"]), golden_traj["cfg4p_dt"])
    assert np.array_equal(P, golden_traj["cfg4p_q"])


def test_amr_mesh_matches_reference_forest():
    cfg = cf.CONFIGS["cfg5"].with_(cells=9)
    forest = spacetree.FaceForest(cf.amr_cells(cfg), 2, True)
    ref = json.load(open(os.path.join(GOLDEN, "mesh_cfg5_proxy.json")))
    assert [[l, list(ix)] for l, ix in forest.sfc] == ref["sfc"]
    mine = list(forest.faces.values())
    assert len(mine) == len(ref["faces"])
    for f, r in zip(mine, ref["faces"]):
        assert [f.axis, f.level, list(f.pos)] == r["key"]
        tags = [("virtual" if s == "virtual" else s) for s in f.sides]
        assert tags == r["sides"]
        assert [None if o is None else [o[0], list(o[1])] for o in f.owners] == r["owners"]
        assert len(f.children or ()) == r["children"]
        assert (None if f.child_pos is None else list(f.child_pos)) == r["child_pos"]
        assert (None if f.parent is None else [f.parent.axis, f.parent.level, list(f.parent.pos)]) == r["parent"]
    skel = [[l, list(ix)] for l, ix in forest.sfc if forest.is_skeleton_amr((l, ix))]
    assert skel == ref["skeleton"]


def test_amr_proxy_trajectory(golden_traj):
    cfg = cf.CONFIGS["cfg5"].with_(cells=9)
    forest = spacetree.FaceForest(cf.amr_cells(cfg), 2, True)
    Q0 = cf.initial_dg_amr(cfg, forest.sfc)
    assert np.array_equal(Q0, golden_traj["cfg5p_q0"])
    Q, log = drivers.dg_amr_run(forest, {k: Q0[i] for i, k in enumerate(forest.sfc)}, ops.euler(2),
                                cfg.order, cfg.cfl, 3)
    assert np.array_equal(np.array(log["dt"]), golden_traj["cfg5p_dt"])
    assert np.array_equal(np.stack(log["iterations"]), golden_traj["cfg5p_its"])
    assert np.array_equal(np.stack([Q[k] for k in forest.sfc]), golden_traj["cfg5p_q"])


def test_amr_conservation():
    # periodic AMR run conserves sum of integral(Q)
    cfg = cf.CONFIGS["cfg5"].with_(cells=9)
    forest = spacetree.FaceForest(cf.amr_cells(cfg), 2, True)
    Q0 = cf.initial_dg_amr(cfg, forest.sfc)
    b = ops.basis_for(cfg.order)
    w2 = np.outer(b.weights, b.weights)

    def mass(Q):
        return sum((Q[k] * w2).sum(axis=(1, 2)) * (3.0 ** -k[0]) ** 2 for k in forest.sfc)

    Qd = {k: Q0[i] for i, k in enumerate(forest.sfc)}
    m0 = mass(Qd)
    Q, _ = drivers.dg_amr_run(forest, Qd, ops.euler(2), cfg.order, cfg.cfl, 2)
    assert np.abs(mass(Q) - m0).max() / np.abs(m0).max() < 1e-13


@pytest.mark.parametrize("name", ["deep2d", "deep3d"])
def test_deep_chain_forest_matches_reference(name):
    """Multi-level hanging-face chains (mesh.py:67-100, 355-424): the oracle
    face forest equals the reference Mesh's on meshes with two-level jumps
    between face neighbours (tests/golden/make_golden_deep.py)."""
    ref = json.load(open(os.path.join(GOLDEN, "mesh_deep.json")))[name]
    cells = [(l, tuple(ix)) for l, ix in ref["sfc"]]
    forest = spacetree.FaceForest(cells, ref["dim"], ref["periodic"])
    assert [[l, list(ix)] for l, ix in forest.sfc] == ref["sfc"]
    mine = {tuple([f.axis, f.level, tuple(f.pos)]): f for f in forest.faces.values()}
    assert len(mine) == len(ref["faces"])
    deep = 0
    for r in ref["faces"]:
        f = mine[(r["key"][0], r["key"][1], tuple(r["key"][2]))]
        assert list(f.sides) == r["sides"]
        assert [None if o is None else [o[0], list(o[1])] for o in f.owners] == r["owners"]
        assert len(f.children or ()) == r["children"]
        assert (None if f.child_pos is None else list(f.child_pos)) == r["child_pos"]
        assert (None if f.parent is None else [f.parent.axis, f.parent.level, list(f.parent.pos)]) == r["parent"]
        deep += f.parent is not None and f.parent.parent is not None
    assert deep > 0                                  # the mesh really has two-level chains
    skel = [[l, list(ix)] for l, ix in forest.sfc if forest.is_skeleton_amr((l, ix))]
    assert skel == ref["skeleton"]


@pytest.mark.parametrize("name", ["deep2d", "deep3d"])
def test_deep_chain_oracle_conserves(name):
    """The multi-level restriction is the L2 adjoint of the interpolation at
    every level, so a periodic (2-D) run conserves every component's integral
    and a 3-D outflow run stays finite and matches its two-step rerun."""
    ref = json.load(open(os.path.join(GOLDEN, "mesh_deep.json")))[name]
    cells = [(l, tuple(ix)) for l, ix in ref["sfc"]]
    dim = ref["dim"]
    forest = spacetree.FaceForest(cells, dim, ref["periodic"])
    p = 2
    rng = np.random.default_rng(5)
    Q = {}
    for k in forest.sfc:
        q = np.empty((dim + 2,) + (p + 1,) * dim)
        q[0] = 1.0 + 0.1 * rng.random(q.shape[1:])
        for i in range(dim):
            q[1 + i] = q[0] * (0.3 + 0.1 * rng.random(q.shape[1:]))
        q[1 + dim] = 2.5 + 0.5 * sum(q[1 + i] ** 2 for i in range(dim)) / q[0]
        Q[k] = q
    b = ops.basis_for(p)
    w = fullrun_tensor(b.weights, dim)

    def mass(Qd):
        return sum((Qd[k] * w).reshape(dim + 2, -1).sum(axis=1) * (3.0 ** -k[0]) ** dim for k in forest.sfc)

    Qn, log = drivers.dg_amr_run(forest, Q, ops.euler(dim), p, 0.2, 3)
    assert all(np.isfinite(v).all() for v in Qn.values())
    if ref["periodic"]:
        assert np.allclose(mass(Qn), mass(Q), rtol=1e-13, atol=1e-15)


def fullrun_tensor(w, dim):
    out = w
    for _ in range(dim - 1):
        out = np.multiply.outer(out, w)
    return out
