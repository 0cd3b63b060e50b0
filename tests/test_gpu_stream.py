"""Slab-streamed host steps (DGSolver.step_host): host state in, host state
out, uploads / predictor / corrector / downloads overlapped per slab.  The
result must be bitwise that of set_state(q_in); step() -- every cell's
predictor and corrector are cell-local and the dt minimum is order-free --
for periodic and outflow grids, any slab count, and back-to-back calls whose
input is the previous call's output buffer."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def edg():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1806_07984_b200 as pkg
    return pkg


def _solver(edg, cfg, N):
    pde = edg.pde.make_pde(cfg.pde, dim=cfg.dim, **({"velocity": cfg.velocity} if cfg.pde == "advection" else {}))
    return edg.solver.DGSolver(pde, cfg.order, edg.mesh.CartesianMesh(N, cfg.dim, cfg.periodic), cfg.cfl)


def _initial(edg, cfg, N):
    c = cfg.with_(cells=N)
    return edg.configs.initial_dg_uniform(c)


# slabs = None: the slab count step_host picks from the state size (one slab
# for these small states; cfg3 at 24^3 is 69 MB -> 16 slabs)
@pytest.mark.parametrize("tag,N,slabs", [("cfg2", 12, 1), ("cfg2", 12, 5), ("cfg2", 12, 12), ("cfg3", 8, 3),
                                         ("cfg3", 8, 8), ("cfg1", 27, 16), ("cfg1", 27, None), ("cfg2", 12, None),
                                         ("cfg3", 24, None)])
def test_step_host_bitwise_vs_step(edg, tag, N, slabs):
    import torch
    cfg = edg.configs.CONFIGS[tag]
    if tag == "cfg2":
        cfg = cfg.with_(cfl=0.2)
    Q0 = _initial(edg, cfg, N)
    steps = 3
    ref = _solver(edg, cfg, N)
    ref.set_state(Q0)
    ref.run(steps, graph=False)
    ref.check_status()
    want = ref.state().cpu().numpy()
    want_dt = ref.dt_history()

    s = _solver(edg, cfg, N)
    a = torch.from_numpy(np.ascontiguousarray(Q0)).pin_memory()
    b = torch.empty_like(a).pin_memory()
    s.set_state(a)          # (the solver's own first state; step_host overwrites it)
    s.steps_done = 0
    for _ in range(steps):
        s.step_host(a, b, slabs=slabs)
        a, b = b, a
    s.host_wait()
    torch.cuda.synchronize()
    s.check_status()
    assert np.array_equal(a.numpy(), want)
    assert np.array_equal(s.state().cpu().numpy(), want)
    assert np.array_equal(s.dt_history(), want_dt)


def test_step_host_after_device_steps(edg):
    """step_host after eager device steps on the same solver (the uploads wait
    for the device work), then device steps again from its result."""
    import torch
    cfg = edg.configs.CONFIGS["cfg3"]
    N = 6
    Q0 = _initial(edg, cfg, N)
    ref = _solver(edg, cfg, N)
    ref.set_state(Q0)
    ref.run(4, graph=False)
    want = ref.state().cpu().numpy()

    s = _solver(edg, cfg, N)
    s.set_state(Q0)
    s.step()
    mid = s.state().cpu().numpy()
    a = torch.from_numpy(mid).pin_memory()
    b = torch.empty_like(a).pin_memory()
    s.step_host(a, b, slabs=4)
    s.host_wait()
    s.run(2, graph=False)
    torch.cuda.synchronize()
    assert np.array_equal(s.state().cpu().numpy(), want)


def test_step_host_rejects_adaptive(edg):
    from paper_1806_07984_b200.errors import ConfigError
    mesh = edg.mesh.AdaptiveMesh([(1, (i, j)) for i in range(3) for j in range(3)], 2, True)
    s = edg.solver.DGSolver(edg.pde.euler(2), 3, mesh, 0.2)
    with pytest.raises(ConfigError):
        s.step_host(None, None)



@pytest.mark.parametrize("cells,slabs", [(16, 1), (16, 2), (32, 3), (32, 4)])
def test_fv_step_host_bitwise_vs_step(edg, cells, slabs):
    """Config 4's patch update streamed from / to host buffers in slabs of
    patch layers: bitwise the device step (which is bitwise the reference)."""
    import torch
    cfg = edg.configs.CONFIGS["cfg4"].with_(cells=cells)
    P0 = edg.configs.initial_fv(cfg)
    ref = edg.solver.FVSolver(edg.pde.euler(3), cells, 8, cfg.cfl)
    ref.set_state(P0)
    ref.run(3, graph=False)
    want = ref.state().cpu().numpy()
    s = edg.solver.FVSolver(edg.pde.euler(3), cells, 8, cfg.cfl)
    a = torch.from_numpy(np.ascontiguousarray(P0)).pin_memory()
    b = torch.empty_like(a).pin_memory()
    for _ in range(3):
        s.step_host(a, b, slabs=slabs)
        a, b = b, a
    s.host_wait()
    torch.cuda.synchronize()
    s.check_status()
    assert np.array_equal(a.numpy(), want)
    assert np.array_equal(s.dt_history(), ref.dt_history())
