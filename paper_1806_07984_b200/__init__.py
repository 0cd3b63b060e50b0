"""enclavedg_b200 -- B200-native (sm_100a) ADER-DG cell/face hot path.

Drop-in for the operator API of the reference package `enclavedg`
(arXiv 1806.07984): stp_picard, riemann_rusanov, corrector, fv_patch_update,
patch_boundary_layers, admissible_dt, project_to_faces, the 3:1 face transfer,
plus GPU time-step drivers (solver.DGSolver / solver.FVSolver) that replace
the Algorithm-1 loop and the enclave task runtime with a two-priority-stream
CUDA schedule.  All compute runs in libenclavedg_b200.so (hand-written fp64
CUDA for sm_100a) through the C ABI in include/enclavedg_b200.h.
"""
from . import errors, configs, basis, pde, _lib, kernels, transfer, mesh, solver, decomposition, sharded, io  # noqa: F401

__all__ = ["errors", "configs", "basis", "pde", "kernels", "transfer", "mesh", "solver", "decomposition", "sharded", "io"]
