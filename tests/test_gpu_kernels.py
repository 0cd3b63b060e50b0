"""GPU parity of the per-kernel C-ABI entry points against the golden vectors
produced by the reference package (tests/golden/ops.npz) and the oracle."""
import numpy as np
import pytest

from conftest import rel_linf

pytestmark = pytest.mark.gpu

PDES = {0: "advection", 1: "burgers", 2: "euler"}


@pytest.fixture(scope="module")
def edg():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1806_07984_b200 as pkg
    from paper_1806_07984_b200 import _lib
    _lib.load()
    return pkg


def _pde(pkg, code, dim):
    if PDES[code] == "advection":
        return pkg.pde.advection(velocity=(1.0, 0.5, 0.25)[:dim], dim=dim)
    return pkg.pde.make_pde(PDES[code], dim=dim)


def _keys(dim):
    return [(a, s) for a in range(dim) for s in (0, 1)]


@pytest.mark.parametrize("ci", range(8))
def test_stp_picard_vs_reference_vectors(edg, golden_ops, ci):
    import torch
    g = lambda k: golden_ops[f"stp{ci}_{k}"]  # noqa: E731
    dim, p, code = (int(v) for v in g("meta"))
    pde = _pde(edg, code, dim)
    b = edg.basis.get_basis(p)
    Q = torch.from_numpy(g("q")).cuda()
    r = edg.kernels.stp_picard_batch(Q, pde, float(g("dt")), b, tuple(g("edges")))
    torch.cuda.synchronize()
    assert np.array_equal(r["iterations"].cpu().numpy(), g("iterations"))
    assert np.array_equal(r["converged"].cpu().numpy().astype(bool), g("converged"))
    # fp64 contraction order differs from OpenBLAS: a few ULP per operation
    assert rel_linf(r["q_end"].cpu().numpy(), g("q_end")) < 1e-12
    assert rel_linf(r["q_int"].cpu().numpy(), g("q_int")) < 1e-12
    assert rel_linf(r["trace_q"].cpu().numpy(), g("trace_q")) < 1e-12
    assert rel_linf(r["trace_f"].cpu().numpy(), g("trace_f")) < 1e-12


def test_stp_picard_single_cell_api(edg, golden_ops):
    g = lambda k: golden_ops[f"stp1_{k}"]  # noqa: E731
    pde = edg.pde.euler(2)
    b = edg.basis.get_basis(5)
    st = edg.kernels.stp_picard(g("q")[0], pde, float(g("dt")), b, tuple(g("edges")))
    assert isinstance(st.q_end, np.ndarray)
    assert st.iterations == g("iterations")[0] and st.converged == bool(g("converged")[0])
    for j, k in enumerate(_keys(2)):
        assert rel_linf(st.trace_f[k], g("trace_f")[0, j]) < 1e-12


def test_corrector_bitwise(edg, golden_ops):
    for ci in range(8):
        g = lambda k: golden_ops[f"stp{ci}_{k}"]  # noqa: E731
        dim, p, code = (int(v) for v in g("meta"))
        b = edg.basis.get_basis(p)
        keys = _keys(dim)
        for c in range(g("q").shape[0]):
            store = edg.kernels.PredictorStore(g("q_int")[c], g("q_end")[c],
                                               {k: g("trace_q")[c, j] for j, k in enumerate(keys)},
                                               {k: g("trace_f")[c, j] for j, k in enumerate(keys)})
            outc = {k: g("outcomes")[c, j] for j, k in enumerate(keys)}
            q = edg.kernels.corrector(store, outc, b, tuple(g("edges")))
            assert np.array_equal(q, g("corrected")[c]), (ci, c)
        with pytest.raises(AssertionError):
            edg.kernels.corrector(store, {}, b, tuple(g("edges")))


def test_riemann_bitwise(edg, golden_ops):
    for ci, code, dim, axis in golden_ops["riem_index"]:
        key = f"riem{ci}_{axis}_"
        pde = _pde(edg, int(code), int(dim))
        lo, hi = golden_ops[key + "lo"], golden_ops[key + "hi"]
        for c in range(lo.shape[0]):
            assert np.array_equal(edg.kernels.riemann_rusanov(lo[c], hi[c], pde, int(axis)), golden_ops[key + "out"][c])
            assert np.array_equal(edg.kernels.riemann_rusanov(lo[c], hi[c], pde, int(axis), sign=-1),
                                  golden_ops[key + "neg"][c])


def test_spec_known_answers(edg, golden_ops):
    adv = edg.pde.advection()
    assert np.all(edg.kernels.riemann_rusanov(np.full((1, 4), 2.0), np.full((1, 4), 2.0), adv, 0) == 2.0)
    assert np.all(edg.kernels.riemann_rusanov(np.full((1, 4), 1.0), np.full((1, 4), 0.0), adv, 0) == 1.0)
    assert np.all(edg.kernels.riemann_rusanov(np.full((1, 4), 2.0), np.full((1, 4), 0.0), edg.pde.burgers(), 0) == 3.0)
    mesh = edg.mesh.CartesianMesh(9, 2, True)
    cells = [((2, (0, 0)), np.ones((1, 4, 4))) for _ in range(81)]
    dt = edg.kernels.admissible_dt(cells, edg.pde.advection((1.0, 0.0)), 3, 0.9, mesh)
    assert dt == float(golden_ops["kat_dt_adv_h9"])


def test_admissible_dt_nan_and_zero(edg, golden_ops):
    Q = golden_ops["dt_euler_q"]

    class M:
        dim = 2

        @staticmethod
        def cell_edges(level):
            return (1 / 9, 1 / 9)

    dt = edg.kernels.admissible_dt([((2, (0, 0)), Q[c]) for c in range(Q.shape[0])], edg.pde.euler(2), 3, 0.9, M)
    assert dt == float(golden_ops["dt_euler_val"])
    zero = np.zeros((4, 4, 4))
    zero[0] = 1.0
    with pytest.raises(edg.errors.EnclaveDgError):
        edg.kernels.admissible_dt([((2, (0, 0)), zero)], edg.pde.euler(2), 3, 0.9, M)


@pytest.mark.parametrize("ci", range(3))
def test_fv_patch_bitwise(edg, golden_ops, ci):
    key = f"fv{ci}_"
    dim, k, code = (int(v) for v in golden_ops[key + "meta"])
    pde = _pde(edg, code, dim)
    P, H = golden_ops[key + "patch"], golden_ops[key + "halos"]
    dt = float(golden_ops[key + "dt"])
    for c in range(P.shape[0]):
        halos = {kk: H[c, j] for j, kk in enumerate(_keys(dim))}
        assert np.array_equal(edg.kernels.fv_patch_update(P[c], pde, dt, (1 / 16,) * dim, halos),
                              golden_ops[key + "out"][c])
        lay = edg.kernels.patch_boundary_layers(P[c])
        for j, kk in enumerate(_keys(dim)):
            assert np.array_equal(lay[kk], golden_ops[key + "layers"][c, j])
    with pytest.raises(edg.errors.NotReadyError):
        edg.kernels.fv_patch_update(P[0], pde, dt, (1 / 16,) * dim, {})


def test_transfer_functions(edg, golden_ops):
    for p in (2, 3, 4):
        t = edg.transfer.get_transfer(p)
        tr2, tr3 = golden_ops[f"xfer{p}_tr2"], golden_ops[f"xfer{p}_tr3"]
        for j in range(3):
            assert rel_linf(edg.transfer.interpolate_face_trace(t, tr2, (j,)), golden_ops[f"xfer{p}_i2_{j}"]) < 1e-15
            assert rel_linf(edg.transfer.restrict_face_values(t, tr2, (j,)), golden_ops[f"xfer{p}_r2_{j}"]) < 1e-15
            for l in range(3):
                assert rel_linf(edg.transfer.interpolate_face_trace(t, tr3, (j, l)),
                                golden_ops[f"xfer{p}_i3_{j}{l}"]) < 1e-15
                assert rel_linf(edg.transfer.restrict_face_values(t, tr3, (j, l)),
                                golden_ops[f"xfer{p}_r3_{j}{l}"]) < 1e-15
        import types
        buf = types.SimpleNamespace(write_guard=None, accum_sweep=None, outcome=None, restricted_children=set())
        for j in range(3):
            edg.transfer.restrict_riemann(t, buf, tr2 * (j + 1), (j,), 7)
        assert rel_linf(buf.outcome, golden_ops[f"xfer{p}_acc2"]) < 1e-15
        with pytest.raises(AssertionError):
            edg.transfer.restrict_riemann(t, buf, tr2, (0,), 7)
        with pytest.raises(edg.errors.NotReadyError):
            edg.transfer.interpolate_to_virtual(t, tr2, (0,), stp_complete=False)


def test_project_to_faces_matches_oracle(edg):
    from oracle import ops
    rng = np.random.default_rng(5)
    for dim, p in ((2, 5), (3, 4), (2, 3)):
        q = rng.standard_normal((3,) + (p + 1,) * dim)
        mine = edg.kernels.project_to_faces(q, edg.basis.get_basis(p))
        ref = ops.face_traces(q, ops.basis_for(p))
        for k in ref:
            assert rel_linf(mine[k], ref[k]) < 1e-15


def test_unsupported_order_is_config_error(edg):
    """Orders outside the reference's [1, 7] (basis.py:13-14) are a ConfigError,
    on the host (basis) and at the C ABI (edg_supported)."""
    for p in (0, 8):
        with pytest.raises(edg.errors.ConfigError):
            edg.basis.get_basis(p)
        for dim in (2, 3):
            with pytest.raises(edg.errors.ConfigError):
                edg.kernels._check_supported(edg.pde.euler(dim), p)


def test_grid_and_table_paths_agree_bitwise(edg):
    """The table-driven entry points (edg_corrector with nbr, edg_fv_patch_step
    with nbr) and the index-arithmetic ones the solvers use give identical bits."""
    import torch
    cfg = edg.configs.CONFIGS["cfg3"].with_(cells=6)
    mesh = edg.mesh.CartesianMesh(6, 3, False, extent=6 / 64)
    s = edg.solver.DGSolver(edg.pde.euler(3), cfg.order, mesh, cfg.cfl)
    s.set_state(edg.configs.initial_dg_uniform(edg.configs.CONFIGS["cfg3"], window=(14, 6)))
    s.step()
    torch.cuda.synchronize()
    q_grid = s.state().clone()
    q_tab = edg.kernels.corrector_batch(s.pde, s.basis, s.q_end, s.trace_f, (1 / 64,) * 3,
                                        nbr=s.nbr, trace_q=s.trace_q)
    assert torch.equal(q_grid, q_tab)
    f = edg.solver.FVSolver(edg.pde.euler(3), 16, 8, 0.4)
    P0 = edg.configs.initial_fv(edg.configs.CONFIGS["cfg4"].with_(cells=16))
    f.set_state(P0)
    f.step()
    torch.cuda.synchronize()
    out = edg.kernels.fv_patch_update_batch(torch.from_numpy(P0).cuda(), f.pde, f.dt_hist[0:1], (0.5, 0.5, 0.5),
                                            nbr=f.nbr)
    assert torch.equal(out, f.state())


def test_stp_linear_vs_reference_ck_vectors(edg, golden_ops):
    """stp_linear (kernels.py:82-106) against the reference's CK outputs."""
    for ci in (0, 5):
        g = lambda k: golden_ops[f"stp{ci}_{k}"]  # noqa: E731
        dim, p, code = (int(v) for v in g("meta"))
        pde = edg.pde.advection((1.0, 0.5, 0.25)[:dim], dim)
        for c in range(g("q").shape[0]):
            st = edg.kernels.stp_linear(g("q")[c], pde, float(g("dt")), edg.basis.get_basis(p), tuple(g("edges")))
            assert rel_linf(st.q_end, g("ck_q_end")[c]) < 1e-12
            assert rel_linf(st.q_int, g("ck_q_int")[c]) < 1e-12
    with pytest.raises(edg.errors.EnclaveDgError):
        edg.kernels.stp_linear(np.ones((4, 4, 4)), edg.pde.euler(2), 1e-3, edg.basis.get_basis(3), (0.1, 0.1))


@pytest.mark.parametrize("n", [1, 31, 729, 59049])
def test_order_by_iterations_is_descending_permutation(edg, n):
    """edg_order_by_iterations (counting sort of the cells by their last
    Picard count, heaviest first): a permutation, counts non-increasing,
    counts >= 63 share the last bucket."""
    import torch
    from paper_1806_07984_b200 import _lib
    rng = np.random.default_rng(n)
    its = rng.integers(0, 80, size=n).astype(np.int32)
    its_d = torch.from_numpy(its).cuda()
    order = torch.full((n,), -1, dtype=torch.int32, device="cuda")
    scratch = torch.zeros(128, dtype=torch.int32, device="cuda")
    import ctypes
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for _ in range(2):   # the histogram is left zeroed for the next call
        _lib.check(_lib.load().edg_order_by_iterations(n, _lib.ptr(its_d), _lib.ptr(order), _lib.ptr(scratch), st),
                   "order")
        torch.cuda.synchronize()
        o = order.cpu().numpy()
        assert np.array_equal(np.sort(o), np.arange(n))
        key = np.minimum(its[o], 63)
        assert np.all(np.diff(key) <= 0)
        assert not scratch[:64].any()
