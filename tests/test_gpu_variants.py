"""The two fused Riemann + corrector kernels agree bit for bit.

The uniform-grid step uses the persistent, bulk-copy double-buffered
corrector (`corrector_grid_pipe_kernel`, edg_corr_pipe.cuh) whenever the grid
gives a persistent CTA more than one group of cells; smaller grids and the
neighbour-table entry point (`edg_corrector` with `nbr`) use the
one-CTA-per-group kernel (`corrector_kernel<..., FUSED>`, edg_faces.cuh).  Both
restate kernels.py:162-193 with the same operation order, so on the same
predictor output they must give identical bits, including the next step's dt
candidate.  The grids below are large enough for the pipelined kernel.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _predict(cfg, N):
    import paper_1806_07984_b200 as edg
    cfg = cfg.with_(cells=N)
    pde = edg.pde.make_pde(cfg.pde, dim=cfg.dim)
    mesh = edg.mesh.CartesianMesh(N, cfg.dim, cfg.periodic)
    s = edg.solver.DGSolver(pde, cfg.order, mesh, cfg.cfl)
    s.set_state(edg.configs.initial_dg_uniform(cfg))
    s._finalize_dt()
    edg._lib.check(s._stp(s.work_order, s.ncells), "stp")
    return edg, s


@pytest.mark.parametrize("name,N", [("cfg2", 128), ("cfg3", 20)])
def test_pipelined_corrector_equals_one_cta_per_group(name, N):
    import ctypes as C
    import torch
    edg, s = _predict(edg_cfg(name), N)
    lib = s.lib
    slots_a = torch.empty_like(s.slots)
    slots_b = torch.empty_like(s.slots)
    status = torch.zeros_like(s.status)
    for sl in (slots_a, slots_b):
        edg._lib.check(lib.edg_dt_slots_reset(edg._lib.ptr(sl), edg.kernels._stream()), "reset")
    # pipelined grid kernel (solver path)
    out_a = torch.empty_like(s.Q)
    edg._lib.check(lib.edg_corrector_grid(C.byref(s.native), s.order, edg._lib.ptr(s.table), s.mesh.N,
                                          int(s.mesh.periodic), edg._lib.ptr(s.q_end), edg._lib.ptr(s.trace_q),
                                          edg._lib.ptr(s.trace_f), edg._lib.ptr(s.edges), edg._lib.ptr(out_a),
                                          edg._lib.ptr(slots_a), edg._lib.ptr(s.hmin), edg._lib.ptr(status),
                                          edg.kernels._stream()), "grid corrector")
    # one-CTA-per-group kernel through the neighbour table
    out_b = edg.kernels.corrector_batch(s.pde, s.basis, s.q_end, s.trace_f, [s.mesh.h] * s.pde.dim, nbr=s.nbr,
                                        trace_q=s.trace_q, dt_slots=slots_b, hmin=s.hmin, status=status)
    torch.cuda.synchronize()
    assert torch.equal(out_a, out_b)
    # the CTAs spread their candidates over the 256 slots by block index, so
    # only the minimum (what edg_dt_finalize reads) is comparable
    assert int(slots_a.min()) == int(slots_b.min())
    assert int(status[0].item()) == 0


def edg_cfg(name):
    import paper_1806_07984_b200 as edg
    return edg.configs.CONFIGS[name]
