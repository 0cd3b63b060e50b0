/*
 * enclavedg_b200 -- C ABI of the B200 (sm_100a) ADER-DG cell/face hot path.
 *
 * Drop-in boundary for the operator API of the reference package
 * `enclavedg` (/root/reference/pkg/src/enclavedg).  The reference is pure
 * Python/numpy and has no FFI; each entry point below replaces one reference
 * function (cited file:line) and is what a ctypes/cffi binding of that
 * function binds.  All pointers named *_dev are CUDA
 * device pointers; everything else is host memory.  No torch types cross the
 * boundary.  Every call is asynchronous on `stream` and returns a status.
 *
 * Layouts (reference kernels.py:5-10, component axis first):
 *   cell DoFs   q[c][k][i0][i1][(i2)]        (C, m, n^d), last axis fastest
 *   face traces t[c][2a+s][k][f]             (C, 2d, m, n^(d-1)); face (a, s)
 *               keeps the non-normal axes in order
 *   FV patches  P[b][k][x][y][z]             (B, m, k, k, k)
 *
 * Operators: `basis_dev` is a packed fp64 table built on the host by numpy
 * exactly as the reference builds them (basis.py:34-65, kernels.py:109-114,
 * transfer.py:28-39) and uploaded verbatim, offsets EDG_BASIS_*(n).
 */
#ifndef ENCLAVEDG_B200_H
#define ENCLAVEDG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes: errors.py:4-33 + SPEC.md:581 exit codes ---------------- */
#define EDG_OK 0
#define EDG_ERR_CONFIG 2     /* ConfigError: unsupported order / dim / pde     */
#define EDG_ERR_NUMERICAL 3  /* NumericalError: non-finite state detected      */
#define EDG_ERR_PROTOCOL 4   /* NotReadyError / AssertionError (missing data)  */
#define EDG_ERR_CUDA 5       /* CUDA launch / runtime failure                  */
#define EDG_ERR_NO_SPEED 6   /* EnclaveDgError: no positive wave speed         */

/* ---- PDE plugin (pde.py:10-24); flux / max_eigenvalue are compiled in ----- */
#define EDG_PDE_ADVECTION 0  /* pde.py:27-37 */
#define EDG_PDE_BURGERS 1    /* pde.py:40-49 */
#define EDG_PDE_EULER 2      /* added system */

typedef struct {
  int32_t kind;        /* EDG_PDE_* */
  int32_t dim;         /* 2 or 3 */
  int32_t m;           /* components: 1 (advection, burgers) or dim + 2 */
  int32_t reserved;
  double gamma;        /* Euler ratio of specific heats */
  double velocity[3];  /* advection velocity */
} edg_pde;

/* packed operator table of one order, n = p + 1 nodes (doubles) */
#define EDG_BASIS_D(n) 0                              /* D[i][j] = l_j'(x_i)   */
#define EDG_BASIS_W(n) ((n) * (n))                    /* GL weights on [0,1]   */
#define EDG_BASIS_TL(n) ((n) * (n) + (n))             /* l_j(0)                */
#define EDG_BASIS_TR(n) ((n) * (n) + 2 * (n))         /* l_j(1)                */
#define EDG_BASIS_KINV(n) ((n) * (n) + 3 * (n))       /* K^-1 (kernels.py:109) */
#define EDG_BASIS_KLIFT(n) (2 * (n) * (n) + 3 * (n))  /* K^-1 @ lift           */
#define EDG_BASIS_INTERP(n) (2 * (n) * (n) + 4 * (n)) /* interp[3][n][n]       */
#define EDG_BASIS_RESTR(n) (5 * (n) * (n) + 4 * (n))  /* restrict[3][n][n]     */
#define EDG_BASIS_SIZE(n) (8 * (n) * (n) + 4 * (n))

/* Which (pde, dim, order) instantiations this build carries. */
int edg_supported(const edg_pde* pde, int32_t order);
/* Library version string and the CUDA arch it was compiled for. */
const char* edg_build_info(void);

/* ---- space-time predictor: stp_picard (kernels.py:120-159) --------------
 * Processes the cells cell_list[0..nwork) (or cells 0..nwork) of q.  edges:
 * device [dim] (edges_per_cell = 0) or [ncells][dim] (edges_per_cell = 1).
 * dt_dev: device scalar.  Outputs are written at the cell's own index:
 * q_end, q_int (nullable) (C,m,n^d); trace_q, trace_f (C,2d,m,n^(d-1));
 * iterations (int32), converged (uint8).  max_iter <= 0 selects 2(p+1).
 * iter_total_dev (nullable): += sum of the processed cells' iteration counts
 * (used for algorithmic-flop accounting without a host round trip). */
int edg_stp_picard(const edg_pde* pde, int32_t order, const double* basis_dev,
                   const double* q_dev, const int32_t* cell_list_dev, int32_t nwork,
                   const double* edges_dev, int32_t edges_per_cell, const double* dt_dev,
                   double tol, int32_t max_iter,
                   double* q_end_dev, double* q_int_dev, double* trace_q_dev,
                   double* trace_f_dev, int32_t* iterations_dev, uint8_t* converged_dev,
                   unsigned long long* iter_total_dev, void* stream);

/* Same contract as edg_stp_picard, launched for a background (low-priority)
 * stream: one work block per CTA instead of persistent CTAs, so the CTAs
 * retire as they finish and the high-priority skeleton work of the schedule
 * gets SM slots while this launch is still running. */
int edg_stp_picard_background(const edg_pde* pde, int32_t order, const double* basis_dev,
                   const double* q_dev, const int32_t* cell_list_dev, int32_t nwork,
                   const double* edges_dev, int32_t edges_per_cell, const double* dt_dev,
                   double tol, int32_t max_iter,
                   double* q_end_dev, double* q_int_dev, double* trace_q_dev,
                   double* trace_f_dev, int32_t* iterations_dev, uint8_t* converged_dev,
                   unsigned long long* iter_total_dev, void* stream);

/* ---- stp_linear (kernels.py:82-106): Cauchy-Kowalevski predictor of a
 * linear PDE (advection); other PDEs -> EDG_ERR_NO_SPEED (EnclaveDgError
 * "stp_linear requires a linear flux").  Same buffers as edg_stp_picard;
 * trace_f = F(trace_q) pointwise as in the reference. */
int edg_stp_linear(const edg_pde* pde, int32_t order, const double* basis_dev, const double* q_dev,
                   const int32_t* cell_list_dev, int32_t nwork, const double* edges_dev, int32_t edges_per_cell,
                   const double* dt_dev, double* q_end_dev, double* q_int_dev, double* trace_q_dev,
                   double* trace_f_dev, int32_t* iterations_dev, uint8_t* converged_dev, void* stream);

/* Work ordering for the next predictor launch: order_dev = the cells sorted
 * by descending Picard count (counting sort, 3 small kernels).  scratch_dev:
 * 128 int32, zero-initialised once by the caller. */
int edg_order_by_iterations(int32_t ncells, const int32_t* iterations_dev, int32_t* order_dev,
                            int32_t* scratch_dev, void* stream);

/* ---- project_to_faces (kernels.py:73-79): vol (C,m,n^d) -> (C,2d,m,n^(d-1)) */
int edg_project_to_faces(int32_t dim, int32_t m, int32_t order, const double* basis_dev, int32_t ncells,
                         const double* vol_dev, double* traces_dev, void* stream);

/* ---- riemann_rusanov on face batches (kernels.py:162-173) ----------------
 * lo, hi, out: (nfaces, m, npts); sign >= 0 -> along +axis, else negated. */
int edg_riemann_rusanov(const edg_pde* pde, int32_t nfaces, int32_t npts,
                        const double* lo_dev, const double* hi_dev, int32_t axis,
                        int32_t sign, double* out_dev, void* stream);

/* ---- corrector (kernels.py:176-193) ---------------------------------------
 * Generic form: side_face[c][2a+s] indexes outcomes (F, m, n^(d-1));
 * a negative index is a missing outcome (EDG_ERR_PROTOCOL, reported through
 * status_dev bit 1).  Fused Cartesian form (side_face == NULL): nbr[c][2a+s]
 * is the face neighbour (-1 = outflow ghost, own trace) and the Rusanov
 * outcome is evaluated inline (Riemann is exactly antisymmetric,
 * kernels.py:165-173, so each face's two evaluations agree bitwise).
 * Optionally fuses the next step's admissible-dt candidates
 * (kernels.py:267-281) into dt_slots_dev (EDG_DT_SLOTS uint64 bit patterns,
 * see edg_dt_finalize) using hmin_dev (per cell, or [1] when
 * edges_per_cell == 0), and counts cells with a non-finite result in
 * status_dev[1]. */
#define EDG_DT_SLOTS 256
int edg_corrector(const edg_pde* pde, int32_t order, const double* basis_dev, int32_t ncells,
                  const double* q_end_dev, const double* trace_q_dev, const double* trace_f_dev,
                  const int32_t* nbr_dev, const int32_t* side_face_dev, const double* outcomes_dev,
                  const double* edges_dev, int32_t edges_per_cell,
                  double* q_out_dev, unsigned long long* dt_slots_dev, const double* hmin_dev,
                  uint32_t* status_dev, void* stream);

/* Fused Cartesian corrector on a uniform row-major cells_per_axis^dim grid
 * (periodic or outflow): neighbours by index arithmetic, no table. */
int edg_corrector_grid(const edg_pde* pde, int32_t order, const double* basis_dev, int32_t cells_per_axis,
                       int32_t periodic, const double* q_end_dev, const double* trace_q_dev,
                       const double* trace_f_dev, const double* edges_dev, double* q_out_dev,
                       unsigned long long* dt_slots_dev, const double* hmin_dev, uint32_t* status_dev,
                       void* stream);

/* The same on the cells [cell_begin, cell_begin + cell_count) of the grid
 * (cell_count < 0: to the end).  Neighbour traces are read wherever they lie,
 * so the predictor outputs of the adjacent cells must be complete; used by the
 * slab-streamed host step (solver.DGSolver.step_host), which corrects slab j
 * as soon as the predictor of slab j + 1 is done. */
int edg_corrector_grid_range(const edg_pde* pde, int32_t order, const double* basis_dev, int32_t cells_per_axis,
                             int32_t periodic, int32_t cell_begin, int32_t cell_count, const double* q_end_dev,
                             const double* trace_q_dev, const double* trace_f_dev, const double* edges_dev,
                             double* q_out_dev, unsigned long long* dt_slots_dev, const double* hmin_dev,
                             uint32_t* status_dev, void* stream);

/* ---- admissible_dt (kernels.py:267-281) -----------------------------------
 * edg_cell_speed_reduce: per-cell lambda (max over axes of max over nodes,
 * NaN axes dropped like Python max) -> candidate h_c / ((2p+1) lambda_c) for
 * cells with lambda > 0, min-reduced into dt_slots_dev.  `order` = p (0 for
 * FV).  For FV patches pass npts = k^3 and q as (B, m, npts).
 * edg_dt_finalize: dt = cfl * min(slots); writes dt_dev (and, when
 * dt_hist_dev is non-null, dt_hist_dev[step] -- or, for step < 0,
 * dt_hist_dev[status_dev[2]++] bounded by -step), re-arms the slots; no
 * positive speed -> dt = NaN and status_dev[0] |= 1 (EDG_ERR_NO_SPEED).
 * status_dev layout: [0] flags, [1] non-finite cell results (cumulative),
 * [2] step counter, [3] first step (1-based) whose result was non-finite. */
int edg_cell_speed_reduce(const edg_pde* pde, int32_t order, int32_t ncells, int32_t npts,
                          const double* q_dev, const double* hmin_dev, int32_t h_per_cell,
                          unsigned long long* dt_slots_dev, void* stream);
int edg_dt_slots_reset(unsigned long long* dt_slots_dev, void* stream);
int edg_dt_finalize(unsigned long long* dt_slots_dev, double cfl, double* dt_dev,
                    double* dt_hist_dev, int32_t step, uint32_t* status_dev, void* stream);

/* ---- hanging faces (transfer.py:59-96) -------------------------------------
 * edg_faces_rusanov: leaf faces f with axis[f], side cells cell[f][2],
 * side kinds kind[f][2] (0 cell, 1 virtual = coarse owner's trace
 * interpolated with interp[child_pos], 2 boundary = copy of the other side),
 * child_pos[f][2] transverse digits.  Writes outcomes[f] (m, n^(d-1)).
 * edg_faces_restrict: parent p accumulates, in child order,
 * restrict[child_pos]-contracted outcomes of its 3^(d-1) children
 * (children[p][j] face indices) into outcomes[parent_face[p]]. */
int edg_faces_rusanov(const edg_pde* pde, int32_t order, const double* basis_dev, int32_t nfaces,
                      const int32_t* axis_dev, const int32_t* cell_dev, const int8_t* kind_dev,
                      const int8_t* child_pos_dev, const double* trace_q_dev, double* outcomes_dev,
                      void* stream);
/* Multi-level hanging-face chains (mesh.py:67-100, 355-424): as
 * edg_faces_rusanov, with each leaf's virtual side interpolated from the
 * coarse owner's trace along a chain of vdepth[f] levels; vpath is
 * [F][max_depth][2] int8 transverse digits, coarsest level first
 * (edg_faces_rusanov is the max_depth = 1 case). */
int edg_faces_rusanov_chain(const edg_pde* pde, int32_t order, const double* basis_dev, int32_t nfaces,
                            const int32_t* axis_dev, const int32_t* cell_dev, const int8_t* kind_dev,
                            const int8_t* vpath_dev, const int8_t* vdepth_dev, int32_t max_depth,
                            const double* trace_q_dev, double* outcomes_dev, void* stream);
int edg_faces_restrict(int32_t dim, int32_t m, int32_t order, const double* basis_dev,
                       int32_t nparents, const int32_t* parent_face_dev, const int32_t* children_dev,
                       const int8_t* child_pos_dev, double* outcomes_dev, void* stream);
/* interpolate_face_trace / restrict_face_values on batches (m, n^(d-1)). */
int edg_interpolate_face_trace(int32_t dim, int32_t m, int32_t order, const double* basis_dev,
                               int32_t nfaces, const double* trace_dev, const int8_t* child_pos_dev,
                               int32_t restrict_mode, double* out_dev, void* stream);

/* ---- finite volume: fv_patch_update (kernels.py:225-253) -------------------
 * edg_fv_patch_update: per-patch API, halos (B, 2d, m, k^(d-1)) given.
 * edg_fv_patch_step: patches of a Cartesian patch grid; halos are read from
 * face-neighbour patches nbr[b][2a+s] (-1 = outflow: own boundary layer,
 * kernels.py:256-264).  Optionally fuses the next step's dt candidates.
 * edges: patch extent per axis (device [dim]). */
int edg_fv_patch_update(const edg_pde* pde, int32_t k, int32_t npatches, const double* patch_dev,
                        const double* halos_dev, const double* dt_dev, const double* edges_dev,
                        double* out_dev, void* stream);
int edg_fv_patch_step(const edg_pde* pde, int32_t k, int32_t npatches, const double* patch_dev,
                      const int32_t* nbr_dev, const double* dt_dev, const double* edges_dev,
                      double* out_dev, unsigned long long* dt_slots_dev, double h_cell,
                      uint32_t* status_dev, void* stream);
/* FV step on a row-major patches_per_axis^d patch grid (periodic or
 * outflow): neighbour patches by index arithmetic, no table. */
int edg_fv_grid_step(const edg_pde* pde, int32_t k, int32_t patches_per_axis, int32_t periodic,
                     const double* patch_dev, const double* dt_dev, const double* edges_dev, double* out_dev,
                     unsigned long long* dt_slots_dev, double h_cell, uint32_t* status_dev, void* stream);

/* The same on the patches [patch_begin, patch_begin + patch_count) of the
 * grid (patch_count < 0: to the end); halos are read from the neighbour
 * patches of the input wherever they lie.  One slab of the streamed host step
 * (solver.FVSolver.step_host). */
int edg_fv_grid_step_range(const edg_pde* pde, int32_t k, int32_t patches_per_axis, int32_t periodic,
                           int32_t patch_begin, int32_t patch_count, const double* patch_dev, const double* dt_dev,
                           const double* edges_dev, double* out_dev, unsigned long long* dt_slots_dev, double h_cell,
                           uint32_t* status_dev, void* stream);
/* patch_boundary_layers (kernels.py:256-264): out (B, 2d, m, k^(d-1)). */
int edg_patch_boundary_layers(int32_t dim, int32_t m, int32_t k, int32_t npatches,
                              const double* patch_dev, double* out_dev, void* stream);

/* ---- cell-local operators of dynamic AMR -----
 * edg_gradient_indicator: transfer.py:136-158 on a batch q (C, m, n^d):
 *   ind[c] = max over axes (a NaN axis dropped) of max |D-contraction|
 *   (NaN-propagating over nodes and components); with verdict_dev != NULL
 *   also the refine (+1) / keep (0) / coarsen (-1) verdict against
 *   refine_tol > coarsen_tol and level_dev[c] (NULL = level 0) in
 *   [min_level, max_level] (evaluate_refinement_criterion).
 * edg_interpolate_volume: transfer.py:99-102; item i maps the parent
 *   q[parent_dev[i]] (NULL: q[i]) onto the child with per-axis digits
 *   digits_dev[i][0..dim-1] (int8 [nitems][3]) -> out (nitems, m, n^d).
 * edg_restrict_volume: transfer.py:105-118; children (P, 3^d, m, n^d) in
 *   row-major digit order -> out (P, m, n^d). */
int edg_gradient_indicator(int32_t dim, int32_t m, int32_t order, const double* basis_dev, int32_t ncells,
                           const double* q_dev, const int32_t* level_dev, double refine_tol, double coarsen_tol,
                           int32_t max_level, int32_t min_level, double* ind_dev, int8_t* verdict_dev,
                           void* stream);
int edg_interpolate_volume(int32_t dim, int32_t m, int32_t order, const double* basis_dev, int32_t nitems,
                           const int32_t* parent_dev, const double* q_dev, const int8_t* digits_dev,
                           double* out_dev, void* stream);
int edg_restrict_volume(int32_t dim, int32_t m, int32_t order, const double* basis_dev, int32_t nparents,
                        const double* children_dev, double* out_dev, void* stream);

/* ---- measurement helper: fp64 FMA throughput probe ----------------------
 * Launches `blocks` x 256 threads, each running 8 independent DFMA chains of
 * `iters` steps (flops = blocks * 256 * 8 * iters * 2).  Time it with events
 * on `stream`; used by bench.py for the FP64 roofline denominator, which
 * MEASURED_PEAKS.json does not carry. */
int edg_probe_fp64(double* sink_dev, int32_t blocks, int32_t iters, void* stream);
/* DMMA (mma.sync m8n8k4 f64) probe: blocks x 8 warps x 4 chains x iters
 * MMAs of 8*8*4 FMAs each (flops = blocks * 8 * 4 * iters * 512). */
int edg_probe_dmma(double* sink_dev, int32_t blocks, int32_t iters, void* stream);

/* ---- stream schedule helpers --------------------------------------------- */
/* Priority range of the device (numerically lower = higher priority). */
int edg_stream_priority_range(int32_t* least, int32_t* greatest);
/* Last CUDA error string of this thread (static storage). */
const char* edg_last_error(void);

/* CUDA graphs that keep per-node stream priorities (the skeleton-first
 * schedule of SPEC.md:403-404 inside a replayed graph).  edg_graph_begin
 * starts a relaxed-mode capture on `stream`; edg_graph_end ends it, writes
 * the priority attribute of each captured kernel node (graph node order, at
 * most max_nodes) and their count, and instantiates the executable graph with
 * cudaGraphInstantiateFlagUseNodePriority into *exec_out. */
int edg_graph_begin(void* stream);
int edg_graph_end(void* stream, void** exec_out, int32_t* node_priority, int32_t max_nodes, int32_t* nkernels);
int edg_graph_launch(void* exec, void* stream);
int edg_graph_destroy(void* exec);

/* Launch trace (SPEC.md:392-400 record_trace; tests/test_gpu_schedule.py):
 * the NEXT traced launch issued by the calling host thread (edg_stp_picard,
 * edg_corrector, edg_corrector_grid, edg_faces_rusanov, edg_faces_restrict,
 * edg_dt_finalize, the edg_fv_* updates) records into slot_dev[0..1]: the
 * global-timer ns of its first CTA start (atomicMin) and of its last CTA exit
 * (atomicMax).  Initialise the slot to {UINT64_MAX, 0}.  Inside a stream
 * capture the slot address is baked into the graph node. */
int edg_trace_next(unsigned long long* slot_dev);

/* ---- rank-boundary trace exchange (host half in
 * decomposition.py; replaces the per-face send_face / receive_face payloads of
 * SPEC.md:425-508 and boundary_face_order mesh.py:613-628) ----------------
 * edg_pack_face_traces: out[j][0] = trace_q[cell[j]][side[j]],
 *   out[j][1] = trace_f[cell[j]][side[j]] (row_len = m*n^(d-1) doubles each;
 *   traces (C, nsides, row_len)); out is the send buffer (nfaces, 2, row_len).
 * edg_unpack_face_traces: ghost[slot[j]] = in[j] (ghost (G, 2, row_len)). */
int edg_pack_face_traces(int32_t nsides, int32_t row_len, int32_t nfaces, const int32_t* cell_dev,
                         const int8_t* side_dev, const double* trace_q_dev, const double* trace_f_dev,
                         double* out_dev, void* stream);
int edg_unpack_face_traces(int32_t row_len, int32_t nfaces, const int32_t* slot_dev, const double* in_dev,
                           double* ghost_dev, void* stream);
/* Row gather / scatter of the sharded step (paper_1806_07984_b200/sharded.py;
 * the send_face / receive_face payload placement of SPEC.md:447-466):
 * gather  dst[j] = src[idx[j]]  (pack: rows of trace_q viewed as
 *          (cells * 2d, m * n^(d-1)), idx = cell * 2d + side slot);
 * scatter dst[idx[j]] = src[j]  (unpack into the ghost rows).
 * Rows are row_len doubles; idx is int64. */
int edg_gather_rows(int32_t row_len, int32_t nrows, const int64_t* idx_dev, const double* src_dev, double* dst_dev,
                    void* stream);
int edg_scatter_rows(int32_t row_len, int32_t nrows, const int64_t* idx_dev, const double* src_dev, double* dst_dev,
                     void* stream);

#ifdef __cplusplus
}
#endif
#endif /* ENCLAVEDG_B200_H */
