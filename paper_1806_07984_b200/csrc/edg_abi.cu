// extern "C" entry points of libenclavedg_b200 (declared in
// include/enclavedg_b200.h).  Validates arguments, maps them onto the
// PDE-specialised launchers of the instantiation units, and reports the
// reference's error contract as status codes (errors.py:4-33).
#include <cstdio>
#include <cstring>
#include <type_traits>

#include "edg_stp.cuh"
#include "edg_faces.cuh"
#include "edg_fv.cuh"
#include "edg_dt.cuh"
#include "edg_amr.cuh"

namespace edg {
#define EDG_DECL_UNIT(name)                                                                                  \
  int unit_##name##_stp(int n, const StpArgs& a, cudaStream_t st);                                           \
  int unit_##name##_stl(int n, const StpArgs& a, cudaStream_t st);                                           \
  int unit_##name##_corr(int n, bool fused, const CorrArgs& a, cudaStream_t st);                             \
  int unit_##name##_faces(int n, const FaceArgs& a, cudaStream_t st);                                        \
  int unit_##name##_speed(int order, int ncells, int npts, const double* q, const double* hmin, int h_per_cell, \
                          unsigned long long* slots, const PdeParams& pp, cudaStream_t st);                  \
  int unit_##name##_riemann(int nfaces, int npts, const double* lo, const double* hi, int axis, int sign,     \
                            double* out, const PdeParams& pp, cudaStream_t st);                              \
  int unit_##name##_fv(int k, const FvArgs& a, cudaStream_t st);                                             \
  int unit_##name##_max_n();
EDG_DECL_UNIT(advection2)
EDG_DECL_UNIT(advection3)
EDG_DECL_UNIT(burgers2)
EDG_DECL_UNIT(burgers3)
EDG_DECL_UNIT(euler2)
EDG_DECL_UNIT(euler3)

struct Unit {
  int (*stp)(int, const StpArgs&, cudaStream_t);
  int (*stl)(int, const StpArgs&, cudaStream_t);
  int (*corr)(int, bool, const CorrArgs&, cudaStream_t);
  int (*faces)(int, const FaceArgs&, cudaStream_t);
  int (*speed)(int, int, int, const double*, const double*, int, unsigned long long*, const PdeParams&, cudaStream_t);
  int (*riemann)(int, int, const double*, const double*, int, int, double*, const PdeParams&, cudaStream_t);
  int (*fv)(int, const FvArgs&, cudaStream_t);
  int (*max_n)();
};
#define EDG_UNIT(name) \
  Unit { unit_##name##_stp, unit_##name##_stl, unit_##name##_corr, unit_##name##_faces, unit_##name##_speed, unit_##name##_riemann, unit_##name##_fv, unit_##name##_max_n }

static const Unit* find_unit(const edg_pde* p) {
  static const Unit units[3][2] = {{EDG_UNIT(advection2), EDG_UNIT(advection3)},
                                   {EDG_UNIT(burgers2), EDG_UNIT(burgers3)},
                                   {EDG_UNIT(euler2), EDG_UNIT(euler3)}};
  if (!p || p->kind < 0 || p->kind > 2 || (p->dim != 2 && p->dim != 3)) return nullptr;
  const int want_m = p->kind == EDG_PDE_EULER ? p->dim + 2 : 1;
  if (p->m != want_m) return nullptr;
  return &units[p->kind][p->dim - 2];
}

static PdeParams params_of(const edg_pde* p) {
  PdeParams pp;
  pp.gamma = p->gamma;
  pp.gm1 = p->gamma - 1.0;
  for (int i = 0; i < 3; ++i) pp.vel[i] = p->velocity[i];
  return pp;
}

static thread_local char g_err[256] = "";
// launch-trace slot for the next traced launch of this host thread (edg_trace_next)
static thread_local unsigned long long* g_trace_next = nullptr;
static unsigned long long* take_trace() {
  unsigned long long* t = g_trace_next;
  g_trace_next = nullptr;
  return t;
}
static int fail(int code, const char* what) {
  std::snprintf(g_err, sizeof g_err, "%s", what);
  return code;
}
static int cuda_status(int code) {
  if (code == EDG_ERR_CUDA) {
    cudaError_t e = cudaGetLastError();
    std::snprintf(g_err, sizeof g_err, "CUDA: %s", cudaGetErrorString(e));
  }
  return code;
}
}  // namespace edg

using namespace edg;

extern "C" {

const char* edg_last_error(void) { return g_err; }

int edg_trace_next(unsigned long long* slot_dev) {
  g_trace_next = slot_dev;
  return EDG_OK;
}

const char* edg_build_info(void) {
  return "enclavedg_b200 1.0 sm_100a fp64 (STP picard / rusanov / corrector / fv / dt / transfer)";
}

int edg_supported(const edg_pde* pde, int32_t order) {
  const Unit* u = find_unit(pde);
  if (!u) return 0;
  return order >= 1 && order + 1 <= u->max_n();
}

}  // extern "C"

static int stp_picard_launch(int ctas_per_sm, const edg_pde* pde, int32_t order, const double* basis_dev, const double* q_dev,
                   const int32_t* cell_list_dev, int32_t nwork, const double* edges_dev, int32_t edges_per_cell,
                   const double* dt_dev, double tol, int32_t max_iter, double* q_end_dev, double* q_int_dev,
                   double* trace_q_dev, double* trace_f_dev, int32_t* iterations_dev, uint8_t* converged_dev,
                   unsigned long long* iter_total_dev, void* stream) {
  unsigned long long* const trace = take_trace();   // consumed even when nothing launches
  const Unit* u = find_unit(pde);
  if (!u) return fail(EDG_ERR_CONFIG, "unsupported pde descriptor");
  if (order < 1 || order + 1 > u->max_n()) return fail(EDG_ERR_CONFIG, "polynomial order not built for this pde/dim");
  if (nwork < 0) return fail(EDG_ERR_CONFIG, "negative work size");
  if (nwork == 0) return EDG_OK;
  if (!basis_dev || !q_dev || !edges_dev || !dt_dev || !q_end_dev || !trace_q_dev || !trace_f_dev ||
      !iterations_dev || !converged_dev)
    return fail(EDG_ERR_CONFIG, "null buffer");
  StpArgs a;
  a.q = q_dev;
  a.cell_list = cell_list_dev;
  a.nwork = nwork;
  a.basis = basis_dev;
  a.edges = edges_dev;
  a.edges_per_cell = edges_per_cell;
  a.dt = dt_dev;
  a.tol = tol;
  a.max_iter = max_iter > 0 ? max_iter : 2 * (order + 1);
  a.pp = params_of(pde);
  a.q_end = q_end_dev;
  a.q_int = q_int_dev;
  a.trace_q = trace_q_dev;
  a.trace_f = trace_f_dev;
  a.iterations = iterations_dev;
  a.converged = converged_dev;
  a.iter_total = iter_total_dev;
  a.trace = trace;
  a.ctas_per_sm = ctas_per_sm;
  return cuda_status(u->stp(order + 1, a, (cudaStream_t)stream));
}

extern "C" {

int edg_stp_picard(const edg_pde* pde, int32_t order, const double* basis_dev, const double* q_dev,
                   const int32_t* cell_list_dev, int32_t nwork, const double* edges_dev, int32_t edges_per_cell,
                   const double* dt_dev, double tol, int32_t max_iter, double* q_end_dev, double* q_int_dev,
                   double* trace_q_dev, double* trace_f_dev, int32_t* iterations_dev, uint8_t* converged_dev,
                   unsigned long long* iter_total_dev, void* stream) {
  return stp_picard_launch(0, pde, order, basis_dev, q_dev, cell_list_dev, nwork, edges_dev, edges_per_cell, dt_dev,
                           tol, max_iter, q_end_dev, q_int_dev, trace_q_dev, trace_f_dev, iterations_dev,
                           converged_dev, iter_total_dev, stream);
}

#ifndef EDG_STP_BACKGROUND_CTAS
#define EDG_STP_BACKGROUND_CTAS (-1)
#endif
int edg_stp_picard_background(const edg_pde* pde, int32_t order, const double* basis_dev, const double* q_dev,
                              const int32_t* cell_list_dev, int32_t nwork, const double* edges_dev,
                              int32_t edges_per_cell, const double* dt_dev, double tol, int32_t max_iter,
                              double* q_end_dev, double* q_int_dev, double* trace_q_dev, double* trace_f_dev,
                              int32_t* iterations_dev, uint8_t* converged_dev, unsigned long long* iter_total_dev,
                              void* stream) {
  return stp_picard_launch(EDG_STP_BACKGROUND_CTAS, pde, order, basis_dev, q_dev, cell_list_dev, nwork, edges_dev,
                           edges_per_cell, dt_dev, tol, max_iter, q_end_dev, q_int_dev, trace_q_dev, trace_f_dev,
                           iterations_dev, converged_dev, iter_total_dev, stream);
}

int edg_stp_linear(const edg_pde* pde, int32_t order, const double* basis_dev, const double* q_dev,
                   const int32_t* cell_list_dev, int32_t nwork, const double* edges_dev, int32_t edges_per_cell,
                   const double* dt_dev, double* q_end_dev, double* q_int_dev, double* trace_q_dev,
                   double* trace_f_dev, int32_t* iterations_dev, uint8_t* converged_dev, void* stream) {
  const Unit* u = find_unit(pde);
  if (!u) return fail(EDG_ERR_CONFIG, "unsupported pde descriptor");
  if (pde->kind != EDG_PDE_ADVECTION) return fail(EDG_ERR_NO_SPEED, "stp_linear requires a linear flux");
  if (order < 1 || order + 1 > u->max_n()) return fail(EDG_ERR_CONFIG, "polynomial order not built for this pde/dim");
  if (nwork <= 0) return EDG_OK;
  StpArgs a;
  std::memset(&a, 0, sizeof a);
  a.q = q_dev;
  a.cell_list = cell_list_dev;
  a.nwork = nwork;
  a.basis = basis_dev;
  a.edges = edges_dev;
  a.edges_per_cell = edges_per_cell;
  a.dt = dt_dev;
  a.pp = params_of(pde);
  a.q_end = q_end_dev;
  a.q_int = q_int_dev;
  a.trace_q = trace_q_dev;
  a.trace_f = trace_f_dev;
  a.iterations = iterations_dev;
  a.converged = converged_dev;
  return cuda_status(u->stl(order + 1, a, (cudaStream_t)stream));
}

int edg_riemann_rusanov(const edg_pde* pde, int32_t nfaces, int32_t npts, const double* lo_dev,
                        const double* hi_dev, int32_t axis, int32_t sign, double* out_dev, void* stream) {
  const Unit* u = find_unit(pde);
  if (!u) return fail(EDG_ERR_CONFIG, "unsupported pde descriptor");
  if (axis < 0 || axis >= pde->dim) return fail(EDG_ERR_CONFIG, "axis out of range");
  return cuda_status(u->riemann(nfaces, npts, lo_dev, hi_dev, axis, sign, out_dev, params_of(pde), (cudaStream_t)stream));
}

int edg_corrector(const edg_pde* pde, int32_t order, const double* basis_dev, int32_t ncells, const double* q_end_dev,
                  const double* trace_q_dev, const double* trace_f_dev, const int32_t* nbr_dev,
                  const int32_t* side_face_dev, const double* outcomes_dev, const double* edges_dev,
                  int32_t edges_per_cell, double* q_out_dev, unsigned long long* dt_slots_dev,
                  const double* hmin_dev, uint32_t* status_dev, void* stream) {
  unsigned long long* const trace = take_trace();   // consumed even when nothing launches
  const Unit* u = find_unit(pde);
  if (!u) return fail(EDG_ERR_CONFIG, "unsupported pde descriptor");
  if (order < 1 || order + 1 > u->max_n()) return fail(EDG_ERR_CONFIG, "polynomial order not built for this pde/dim");
  const bool fused = side_face_dev == nullptr;
  if (fused && (!nbr_dev || !trace_q_dev)) return fail(EDG_ERR_CONFIG, "fused corrector needs nbr and trace_q");
  if (!fused && !outcomes_dev) return fail(EDG_ERR_CONFIG, "generic corrector needs outcomes");
  if (dt_slots_dev && !hmin_dev) return fail(EDG_ERR_CONFIG, "dt fusion needs hmin");
  CorrArgs a;
  a.basis = basis_dev;
  a.ncells = ncells;
  a.cell_base = 0;
  a.order = order;
  a.q_end = q_end_dev;
  a.trace_q = trace_q_dev;
  a.trace_f = trace_f_dev;
  a.nbr = nbr_dev;
  a.grid_n = 0;
  a.periodic = 0;
  a.side_face = side_face_dev;
  a.outcomes = outcomes_dev;
  a.edges = edges_dev;
  a.edges_per_cell = edges_per_cell;
  a.q_out = q_out_dev;
  a.dt_slots = dt_slots_dev;
  a.hmin = hmin_dev;
  a.status = status_dev;
  a.pp = params_of(pde);
  a.trace = trace;
  return cuda_status(u->corr(order + 1, fused, a, (cudaStream_t)stream));
}

int edg_corrector_grid(const edg_pde* pde, int32_t order, const double* basis_dev, int32_t cells_per_axis,
                       int32_t periodic, const double* q_end_dev, const double* trace_q_dev, const double* trace_f_dev,
                       const double* edges_dev, double* q_out_dev, unsigned long long* dt_slots_dev,
                       const double* hmin_dev, uint32_t* status_dev, void* stream) {
  return edg_corrector_grid_range(pde, order, basis_dev, cells_per_axis, periodic, 0, -1, q_end_dev, trace_q_dev,
                                  trace_f_dev, edges_dev, q_out_dev, dt_slots_dev, hmin_dev, status_dev, stream);
}

int edg_corrector_grid_range(const edg_pde* pde, int32_t order, const double* basis_dev, int32_t cells_per_axis,
                             int32_t periodic, int32_t cell_begin, int32_t cell_count, const double* q_end_dev,
                             const double* trace_q_dev, const double* trace_f_dev, const double* edges_dev,
                             double* q_out_dev, unsigned long long* dt_slots_dev, const double* hmin_dev,
                             uint32_t* status_dev, void* stream) {
  unsigned long long* const trace = take_trace();   // consumed even when nothing launches
  const Unit* u = find_unit(pde);
  if (!u) return fail(EDG_ERR_CONFIG, "unsupported pde descriptor");
  if (order < 1 || order + 1 > u->max_n()) return fail(EDG_ERR_CONFIG, "polynomial order not built for this pde/dim");
  if (cells_per_axis < 1 || !trace_q_dev) return fail(EDG_ERR_CONFIG, "grid corrector needs a grid and trace_q");
  if (dt_slots_dev && !hmin_dev) return fail(EDG_ERR_CONFIG, "dt fusion needs hmin");
  long long nc = 1;
  for (int d = 0; d < pde->dim; ++d) nc *= cells_per_axis;
  if (nc > 0x7fffffffLL) return fail(EDG_ERR_CONFIG, "grid too large");
  if (cell_count < 0) cell_count = (int32_t)(nc - cell_begin);
  if (cell_begin < 0 || (long long)cell_begin + cell_count > nc) return fail(EDG_ERR_CONFIG, "cell range outside the grid");
  if (cell_count == 0) return EDG_OK;
  CorrArgs a;
  a.basis = basis_dev;
  a.ncells = cell_begin + cell_count;
  a.cell_base = cell_begin;
  a.order = order;
  a.q_end = q_end_dev;
  a.trace_q = trace_q_dev;
  a.trace_f = trace_f_dev;
  a.nbr = nullptr;
  a.grid_n = cells_per_axis;
  a.periodic = periodic ? 1 : 0;
  a.side_face = nullptr;
  a.outcomes = nullptr;
  a.edges = edges_dev;
  a.edges_per_cell = 0;
  a.q_out = q_out_dev;
  a.dt_slots = dt_slots_dev;
  a.hmin = hmin_dev;
  a.status = status_dev;
  a.pp = params_of(pde);
  a.trace = trace;
  return cuda_status(u->corr(order + 1, true, a, (cudaStream_t)stream));
}

int edg_cell_speed_reduce(const edg_pde* pde, int32_t order, int32_t ncells, int32_t npts, const double* q_dev,
                          const double* hmin_dev, int32_t h_per_cell, unsigned long long* dt_slots_dev, void* stream) {
  const Unit* u = find_unit(pde);
  if (!u) return fail(EDG_ERR_CONFIG, "unsupported pde descriptor");
  return cuda_status(
      u->speed(order, ncells, npts, q_dev, hmin_dev, h_per_cell, dt_slots_dev, params_of(pde), (cudaStream_t)stream));
}

int edg_dt_slots_reset(unsigned long long* dt_slots_dev, void* stream) {
  dt_slots_reset_kernel<<<1, EDG_DT_SLOTS, 0, (cudaStream_t)stream>>>(dt_slots_dev);
  return cuda_status(check_launch());
}

int edg_dt_finalize(unsigned long long* dt_slots_dev, double cfl, double* dt_dev, double* dt_hist_dev, int32_t step,
                    uint32_t* status_dev, void* stream) {
  unsigned long long* const trace = take_trace();   // consumed even when nothing launches
  dt_finalize_kernel<<<1, EDG_DT_SLOTS, 0, (cudaStream_t)stream>>>(dt_slots_dev, cfl, dt_dev, dt_hist_dev, step,
                                                                   status_dev, trace);
  return cuda_status(check_launch());
}

int edg_faces_rusanov_chain(const edg_pde* pde, int32_t order, const double* basis_dev, int32_t nfaces,
                            const int32_t* axis_dev, const int32_t* cell_dev, const int8_t* kind_dev,
                            const int8_t* vpath_dev, const int8_t* vdepth_dev, int32_t max_depth,
                            const double* trace_q_dev, double* outcomes_dev, void* stream) {
  unsigned long long* const trace = take_trace();   // consumed even when nothing launches
  const Unit* u = find_unit(pde);
  if (!u) return fail(EDG_ERR_CONFIG, "unsupported pde descriptor");
  if (order < 1 || order + 1 > u->max_n()) return fail(EDG_ERR_CONFIG, "polynomial order not built for this pde/dim");
  if (max_depth < 1) return fail(EDG_ERR_CONFIG, "chain depth must be >= 1");
  FaceArgs a;
  a.basis = basis_dev;
  a.nfaces = nfaces;
  a.axis = axis_dev;
  a.cell = cell_dev;
  a.kind = kind_dev;
  a.child_pos = vpath_dev;
  a.vdepth = vdepth_dev;
  a.maxd = max_depth;
  a.trace_q = trace_q_dev;
  a.outcomes = outcomes_dev;
  a.pp = params_of(pde);
  a.trace = trace;
  return cuda_status(u->faces(order + 1, a, (cudaStream_t)stream));
}

int edg_faces_rusanov(const edg_pde* pde, int32_t order, const double* basis_dev, int32_t nfaces,
                      const int32_t* axis_dev, const int32_t* cell_dev, const int8_t* kind_dev,
                      const int8_t* child_pos_dev, const double* trace_q_dev, double* outcomes_dev, void* stream) {
  return edg_faces_rusanov_chain(pde, order, basis_dev, nfaces, axis_dev, cell_dev, kind_dev, child_pos_dev, nullptr,
                                 1, trace_q_dev, outcomes_dev, stream);
}

}  // extern "C"

template <int DIM>
static int restrict_dim(int n, const double* basis, int m, int np, const int32_t* pf, const int32_t* ch,
                        const int8_t* cp, double* out, unsigned long long* trace, cudaStream_t st) {
  const long long work = (long long)np * m * ipow(n, DIM - 1);
  if (work <= 0) return EDG_OK;
  const unsigned blocks = (unsigned)((work + 127) / 128);
  switch (n) {
#define EDG_CASE(NN)                                                                         \
  case NN:                                                                                   \
    faces_restrict_kernel<DIM, NN><<<blocks, 128, 0, st>>>(basis, m, np, pf, ch, cp, out, trace); \
    return check_launch();
    EDG_CASE(2) EDG_CASE(3) EDG_CASE(4) EDG_CASE(5) EDG_CASE(6) EDG_CASE(7) EDG_CASE(8)
#undef EDG_CASE
  }
  return EDG_ERR_CONFIG;
}

extern "C" {

int edg_faces_restrict(int32_t dim, int32_t m, int32_t order, const double* basis_dev, int32_t nparents,
                       const int32_t* parent_face_dev, const int32_t* children_dev, const int8_t* child_pos_dev,
                       double* outcomes_dev, void* stream) {
  unsigned long long* const trace = take_trace();   // consumed even when nothing launches
  if (order < 1 || order > 7) return fail(EDG_ERR_CONFIG, "order out of range");
  const cudaStream_t st = (cudaStream_t)stream;
  if (dim == 2)
    return cuda_status(restrict_dim<2>(order + 1, basis_dev, m, nparents, parent_face_dev, children_dev, child_pos_dev,
                                       outcomes_dev, trace, st));
  if (dim == 3)
    return cuda_status(restrict_dim<3>(order + 1, basis_dev, m, nparents, parent_face_dev, children_dev, child_pos_dev,
                                       outcomes_dev, trace, st));
  return fail(EDG_ERR_CONFIG, "dim must be 2 or 3");
}

}  // extern "C"

template <int DIM>
static int transfer_dim(int n, const double* basis, int m, int nf, const double* in, const int8_t* cp, int mode,
                        double* out, cudaStream_t st) {
  const long long work = (long long)nf * m * ipow(n, DIM - 1);
  if (work <= 0) return EDG_OK;
  const unsigned blocks = (unsigned)((work + 127) / 128);
  switch (n) {
#define EDG_CASE(NN)                                                                     \
  case NN:                                                                               \
    face_transfer_kernel<DIM, NN><<<blocks, 128, 0, st>>>(basis, m, nf, in, cp, mode, out); \
    return check_launch();
    EDG_CASE(2) EDG_CASE(3) EDG_CASE(4) EDG_CASE(5) EDG_CASE(6) EDG_CASE(7) EDG_CASE(8)
#undef EDG_CASE
  }
  return EDG_ERR_CONFIG;
}

extern "C" {

int edg_interpolate_face_trace(int32_t dim, int32_t m, int32_t order, const double* basis_dev, int32_t nfaces,
                               const double* trace_dev, const int8_t* child_pos_dev, int32_t restrict_mode,
                               double* out_dev, void* stream) {
  if (order < 1 || order > 7) return fail(EDG_ERR_CONFIG, "order out of range");
  const cudaStream_t st = (cudaStream_t)stream;
  if (dim == 2)
    return cuda_status(transfer_dim<2>(order + 1, basis_dev, m, nfaces, trace_dev, child_pos_dev, restrict_mode,
                                       out_dev, st));
  if (dim == 3)
    return cuda_status(transfer_dim<3>(order + 1, basis_dev, m, nfaces, trace_dev, child_pos_dev, restrict_mode,
                                       out_dev, st));
  return fail(EDG_ERR_CONFIG, "dim must be 2 or 3");
}

}  // extern "C"

template <int DIM>
static int project_dim(int n, const double* basis, int m, int nc, const double* vol, double* out, cudaStream_t st) {
  const long long work = (long long)nc * 2 * DIM * m * ipow(n, DIM - 1);
  if (work <= 0) return EDG_OK;
  const unsigned blocks = (unsigned)((work + 127) / 128);
  switch (n) {
#define EDG_CASE(NN)                                                                  \
  case NN:                                                                            \
    project_faces_kernel<DIM, NN><<<blocks, 128, 0, st>>>(basis, m, nc, vol, out); \
    return check_launch();
    EDG_CASE(2) EDG_CASE(3) EDG_CASE(4) EDG_CASE(5) EDG_CASE(6) EDG_CASE(7) EDG_CASE(8)
#undef EDG_CASE
  }
  return EDG_ERR_CONFIG;
}

extern "C" {

int edg_project_to_faces(int32_t dim, int32_t m, int32_t order, const double* basis_dev, int32_t ncells,
                         const double* vol_dev, double* traces_dev, void* stream) {
  if (order < 1 || order > 7) return fail(EDG_ERR_CONFIG, "order out of range");
  const cudaStream_t st = (cudaStream_t)stream;
  if (dim == 2) return cuda_status(project_dim<2>(order + 1, basis_dev, m, ncells, vol_dev, traces_dev, st));
  if (dim == 3) return cuda_status(project_dim<3>(order + 1, basis_dev, m, ncells, vol_dev, traces_dev, st));
  return fail(EDG_ERR_CONFIG, "dim must be 2 or 3");
}

int edg_fv_patch_update(const edg_pde* pde, int32_t k, int32_t npatches, const double* patch_dev,
                        const double* halos_dev, const double* dt_dev, const double* edges_dev, double* out_dev,
                        void* stream) {
  unsigned long long* const trace = take_trace();   // consumed even when nothing launches
  const Unit* u = find_unit(pde);
  if (!u) return fail(EDG_ERR_CONFIG, "unsupported pde descriptor");
  if (!halos_dev) return fail(EDG_ERR_PROTOCOL, "halo layers missing");
  FvArgs a;
  std::memset(&a, 0, sizeof a);
  a.trace = trace;
  a.npatches = npatches;
  a.patch = patch_dev;
  a.halos = halos_dev;
  a.dt = dt_dev;
  a.edges = edges_dev;
  a.out = out_dev;
  a.pp = params_of(pde);
  return cuda_status(u->fv(k, a, (cudaStream_t)stream));
}

int edg_fv_patch_step(const edg_pde* pde, int32_t k, int32_t npatches, const double* patch_dev,
                      const int32_t* nbr_dev, const double* dt_dev, const double* edges_dev, double* out_dev,
                      unsigned long long* dt_slots_dev, double h_cell, uint32_t* status_dev, void* stream) {
  unsigned long long* const trace = take_trace();   // consumed even when nothing launches
  const Unit* u = find_unit(pde);
  if (!u) return fail(EDG_ERR_CONFIG, "unsupported pde descriptor");
  if (!nbr_dev) return fail(EDG_ERR_PROTOCOL, "patch neighbour table missing");
  FvArgs a;
  std::memset(&a, 0, sizeof a);
  a.trace = trace;
  a.npatches = npatches;
  a.patch = patch_dev;
  a.nbr = nbr_dev;
  a.dt = dt_dev;
  a.edges = edges_dev;
  a.out = out_dev;
  a.dt_slots = dt_slots_dev;
  a.h_cell = h_cell;
  a.status = status_dev;
  a.pp = params_of(pde);
  return cuda_status(u->fv(k, a, (cudaStream_t)stream));
}

int edg_fv_grid_step(const edg_pde* pde, int32_t k, int32_t patches_per_axis, int32_t periodic,
                     const double* patch_dev, const double* dt_dev, const double* edges_dev, double* out_dev,
                     unsigned long long* dt_slots_dev, double h_cell, uint32_t* status_dev, void* stream) {
  return edg_fv_grid_step_range(pde, k, patches_per_axis, periodic, 0, -1, patch_dev, dt_dev, edges_dev, out_dev,
                                dt_slots_dev, h_cell, status_dev, stream);
}

int edg_fv_grid_step_range(const edg_pde* pde, int32_t k, int32_t patches_per_axis, int32_t periodic,
                           int32_t patch_begin, int32_t patch_count, const double* patch_dev, const double* dt_dev,
                           const double* edges_dev, double* out_dev, unsigned long long* dt_slots_dev, double h_cell,
                           uint32_t* status_dev, void* stream) {
  unsigned long long* const trace = take_trace();   // consumed even when nothing launches
  const Unit* u = find_unit(pde);
  if (!u) return fail(EDG_ERR_CONFIG, "unsupported pde descriptor");
  if (patches_per_axis < 1) return fail(EDG_ERR_CONFIG, "empty patch grid");
  long long np = 1;
  for (int d = 0; d < pde->dim; ++d) np *= patches_per_axis;
  if (np > 0x7fffffffLL) return fail(EDG_ERR_CONFIG, "patch grid too large");
  if (patch_count < 0) patch_count = (int32_t)(np - patch_begin);
  if (patch_begin < 0 || (long long)patch_begin + patch_count > np) return fail(EDG_ERR_CONFIG, "patch range outside the grid");
  if (patch_count == 0) return EDG_OK;
  FvArgs a;
  std::memset(&a, 0, sizeof a);
  a.trace = trace;
  a.npatches = patch_begin + patch_count;
  a.patch_base = patch_begin;
  a.patch = patch_dev;
  a.pgrid_n = patches_per_axis;
  a.periodic = periodic ? 1 : 0;
  a.dt = dt_dev;
  a.edges = edges_dev;
  a.out = out_dev;
  a.dt_slots = dt_slots_dev;
  a.h_cell = h_cell;
  a.status = status_dev;
  a.pp = params_of(pde);
  return cuda_status(u->fv(k, a, (cudaStream_t)stream));
}

int edg_patch_boundary_layers(int32_t dim, int32_t m, int32_t k, int32_t npatches, const double* patch_dev,
                              double* out_dev, void* stream) {
  const long long work = (long long)npatches * 2 * dim * m * (dim == 2 ? k : k * k);
  if (work <= 0) return EDG_OK;
  const unsigned blocks = (unsigned)((work + 255) / 256);
  if (dim == 2)
    boundary_layers_kernel<2><<<blocks, 256, 0, (cudaStream_t)stream>>>(m, k, npatches, patch_dev, out_dev);
  else if (dim == 3)
    boundary_layers_kernel<3><<<blocks, 256, 0, (cudaStream_t)stream>>>(m, k, npatches, patch_dev, out_dev);
  else
    return fail(EDG_ERR_CONFIG, "dim must be 2 or 3");
  return cuda_status(check_launch());
}

}  // extern "C"

static __global__ void __launch_bounds__(256) fp64_probe_kernel(double* sink, int iters) {
  double a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = 1.0 + 1e-7 * (threadIdx.x + 37 * k);
  const double b = 0.9999999999, c = 1e-12;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fma(a[k], b, c);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 123.456) sink[0] = s;   // never true; keeps the chains alive
}

// DMMA (mma.sync m8n8k4 f64) throughput probe: 4 independent accumulators per warp
static __global__ void __launch_bounds__(256) dmma_probe_kernel(double* sink, int iters) {
  double a = 1.0 + 1e-9 * threadIdx.x, b = 0.5 - 1e-9 * threadIdx.x;
  double c[4][2];
#pragma unroll
  for (int u = 0; u < 4; ++u) c[u][0] = c[u][1] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
                   : "+d"(c[u][0]), "+d"(c[u][1])
                   : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int u = 0; u < 4; ++u) s += c[u][0] + c[u][1];
  if (s == 123.456) sink[0] = s;
}

extern "C" {

int edg_probe_dmma(double* sink_dev, int32_t blocks, int32_t iters, void* stream) {
  dmma_probe_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(sink_dev, iters);
  return cuda_status(check_launch());
}

int edg_order_by_iterations(int32_t ncells, const int32_t* iterations_dev, int32_t* order_dev,
                            int32_t* scratch_dev, void* stream) {
  if (ncells <= 0) return EDG_OK;
  const cudaStream_t st = (cudaStream_t)stream;
  int32_t* hist = scratch_dev;
  int32_t* offs = scratch_dev + ORDER_BINS;
  const unsigned blocks = (unsigned)((ncells + 255) / 256);
  order_hist_kernel<<<blocks, 256, 0, st>>>(ncells, iterations_dev, hist);
  order_scan_kernel<<<1, 32, 0, st>>>(hist, offs);
  order_scatter_kernel<<<blocks, 256, 0, st>>>(ncells, iterations_dev, offs, order_dev);
  return cuda_status(check_launch());
}

int edg_probe_fp64(double* sink_dev, int32_t blocks, int32_t iters, void* stream) {
  fp64_probe_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(sink_dev, iters);
  return cuda_status(check_launch());
}

int edg_stream_priority_range(int32_t* least, int32_t* greatest) {
  int lo = 0, hi = 0;
  if (cudaDeviceGetStreamPriorityRange(&lo, &hi) != cudaSuccess) return cuda_status(EDG_ERR_CUDA);
  *least = lo;
  *greatest = hi;
  return EDG_OK;
}

// ---- CUDA graphs that keep the stream priorities -------------------------
// A kernel captured from a prioritised stream carries that priority as its
// node's launch attribute; it only takes effect if the executable graph is
// instantiated with cudaGraphInstantiateFlagUseNodePriority (otherwise every
// node runs at the priority of the stream the graph is launched into), which
// torch.cuda.CUDAGraph does not do -- hence these four entry points.
int edg_graph_begin(void* stream) {
  if (cudaStreamBeginCapture((cudaStream_t)stream, cudaStreamCaptureModeRelaxed) != cudaSuccess)
    return cuda_status(EDG_ERR_CUDA);
  return EDG_OK;
}

int edg_graph_end(void* stream, void** exec_out, int32_t* node_priority, int32_t max_nodes, int32_t* nkernels) {
  cudaGraph_t g = nullptr;
  if (cudaStreamEndCapture((cudaStream_t)stream, &g) != cudaSuccess || !g) return cuda_status(EDG_ERR_CUDA);
  size_t n = 0;
  int nk = 0;
  if (cudaGraphGetNodes(g, nullptr, &n) != cudaSuccess) {
    cudaGraphDestroy(g);
    return cuda_status(EDG_ERR_CUDA);
  }
  cudaGraphNode_t* nodes = new cudaGraphNode_t[n > 0 ? n : 1];
  cudaGraphGetNodes(g, nodes, &n);
  for (size_t i = 0; i < n; ++i) {
    cudaGraphNodeType t;
    if (cudaGraphNodeGetType(nodes[i], &t) != cudaSuccess || t != cudaGraphNodeTypeKernel) continue;
    cudaLaunchAttributeValue v;
    std::memset(&v, 0, sizeof v);
    if (cudaGraphKernelNodeGetAttribute(nodes[i], cudaLaunchAttributePriority, &v) != cudaSuccess) v.priority = 0;
    if (node_priority && nk < max_nodes) node_priority[nk] = v.priority;
    ++nk;
  }
  delete[] nodes;
  if (nkernels) *nkernels = nk;
  cudaGraphExec_t ex = nullptr;
  const cudaError_t e = cudaGraphInstantiateWithFlags(&ex, g, cudaGraphInstantiateFlagUseNodePriority);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) return cuda_status(EDG_ERR_CUDA);
  *exec_out = (void*)ex;
  return EDG_OK;
}

int edg_graph_launch(void* exec, void* stream) {
  if (!exec) return fail(EDG_ERR_CONFIG, "null graph");
  if (cudaGraphLaunch((cudaGraphExec_t)exec, (cudaStream_t)stream) != cudaSuccess) return cuda_status(EDG_ERR_CUDA);
  return EDG_OK;
}

int edg_graph_destroy(void* exec) {
  if (exec && cudaGraphExecDestroy((cudaGraphExec_t)exec) != cudaSuccess) return cuda_status(EDG_ERR_CUDA);
  return EDG_OK;
}

}  // extern "C"

// ------------------------------------------- dynamic AMR, cell-local ops --
template <int DIM, typename F>
static int amr_dispatch(int n, F f) {
  switch (n) {
#define EDG_CASE(NN) \
  case NN:           \
    return f(std::integral_constant<int, NN>{});
    EDG_CASE(2) EDG_CASE(3) EDG_CASE(4) EDG_CASE(5) EDG_CASE(6) EDG_CASE(7) EDG_CASE(8)
#undef EDG_CASE
  }
  return EDG_ERR_CONFIG;
}

template <typename K>
static int amr_smem(K kernel, size_t bytes) {
  if (bytes > 48 * 1024 &&
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) != cudaSuccess)
    return EDG_ERR_CUDA;
  return EDG_OK;
}

template <int DIM>
static int indicator_dim(int n, const double* basis, int m, int nc, const double* q, const int32_t* level,
                         double rt, double ct, int maxl, int minl, double* ind, int8_t* verdict, cudaStream_t st) {
  return amr_dispatch<DIM>(n, [&](auto NN) {
    constexpr int N = decltype(NN)::value;
    const size_t bytes = sizeof(double) * (N * N + (size_t)m * ipow(N, DIM));
    auto k = gradient_indicator_kernel<DIM, N>;
    if (amr_smem(k, bytes)) return (int)EDG_ERR_CUDA;
    k<<<nc, kAmrThreads, bytes, st>>>(basis, m, nc, q, level, rt, ct, maxl, minl, ind, verdict);
    return check_launch();
  });
}

template <int DIM>
static int interp_vol_dim(int n, const double* basis, int m, int ni, const int32_t* parent, const double* q,
                          const int8_t* digits, double* out, cudaStream_t st) {
  return amr_dispatch<DIM>(n, [&](auto NN) {
    constexpr int N = decltype(NN)::value;
    const size_t bytes = sizeof(double) * (3 * N * N + 2 * (size_t)m * ipow(N, DIM));
    auto k = interpolate_volume_kernel<DIM, N>;
    if (amr_smem(k, bytes)) return (int)EDG_ERR_CUDA;
    k<<<ni, kAmrThreads, bytes, st>>>(basis, m, ni, parent, q, digits, out);
    return check_launch();
  });
}

template <int DIM>
static int restrict_vol_dim(int n, const double* basis, int m, int np, const double* children, double* out,
                            cudaStream_t st) {
  return amr_dispatch<DIM>(n, [&](auto NN) {
    constexpr int N = decltype(NN)::value;
    const size_t bytes = sizeof(double) * (3 * N * N + 3 * (size_t)m * ipow(N, DIM));
    auto k = restrict_volume_kernel<DIM, N>;
    if (amr_smem(k, bytes)) return (int)EDG_ERR_CUDA;
    k<<<np, kAmrThreads, bytes, st>>>(basis, m, np, children, out);
    return check_launch();
  });
}

extern "C" {

int edg_gradient_indicator(int32_t dim, int32_t m, int32_t order, const double* basis_dev, int32_t ncells,
                           const double* q_dev, const int32_t* level_dev, double refine_tol, double coarsen_tol,
                           int32_t max_level, int32_t min_level, double* ind_dev, int8_t* verdict_dev,
                           void* stream) {
  if (order < 1 || order > 7) return fail(EDG_ERR_CONFIG, "order out of range");
  if (m < 1) return fail(EDG_ERR_CONFIG, "m must be positive");
  // RefinementDecision.__post_init__ (transfer.py:131-133)
  if (verdict_dev && !(refine_tol > coarsen_tol && coarsen_tol >= 0.0))
    return fail(EDG_ERR_CONFIG, "need refine_tol > coarsen_tol >= 0 (hysteresis band)");
  if (ncells <= 0) return EDG_OK;
  const cudaStream_t st = (cudaStream_t)stream;
  if (dim == 2)
    return cuda_status(indicator_dim<2>(order + 1, basis_dev, m, ncells, q_dev, level_dev, refine_tol, coarsen_tol,
                                        max_level, min_level, ind_dev, verdict_dev, st));
  if (dim == 3)
    return cuda_status(indicator_dim<3>(order + 1, basis_dev, m, ncells, q_dev, level_dev, refine_tol, coarsen_tol,
                                        max_level, min_level, ind_dev, verdict_dev, st));
  return fail(EDG_ERR_CONFIG, "dim must be 2 or 3");
}

int edg_interpolate_volume(int32_t dim, int32_t m, int32_t order, const double* basis_dev, int32_t nitems,
                           const int32_t* parent_dev, const double* q_dev, const int8_t* digits_dev,
                           double* out_dev, void* stream) {
  if (order < 1 || order > 7) return fail(EDG_ERR_CONFIG, "order out of range");
  if (m < 1) return fail(EDG_ERR_CONFIG, "m must be positive");
  if (nitems <= 0) return EDG_OK;
  const cudaStream_t st = (cudaStream_t)stream;
  if (dim == 2)
    return cuda_status(interp_vol_dim<2>(order + 1, basis_dev, m, nitems, parent_dev, q_dev, digits_dev, out_dev, st));
  if (dim == 3)
    return cuda_status(interp_vol_dim<3>(order + 1, basis_dev, m, nitems, parent_dev, q_dev, digits_dev, out_dev, st));
  return fail(EDG_ERR_CONFIG, "dim must be 2 or 3");
}

int edg_restrict_volume(int32_t dim, int32_t m, int32_t order, const double* basis_dev, int32_t nparents,
                        const double* children_dev, double* out_dev, void* stream) {
  if (order < 1 || order > 7) return fail(EDG_ERR_CONFIG, "order out of range");
  if (m < 1) return fail(EDG_ERR_CONFIG, "m must be positive");
  if (nparents <= 0) return EDG_OK;
  const cudaStream_t st = (cudaStream_t)stream;
  if (dim == 2) return cuda_status(restrict_vol_dim<2>(order + 1, basis_dev, m, nparents, children_dev, out_dev, st));
  if (dim == 3) return cuda_status(restrict_vol_dim<3>(order + 1, basis_dev, m, nparents, children_dev, out_dev, st));
  return fail(EDG_ERR_CONFIG, "dim must be 2 or 3");
}

}  // extern "C"

// ---- rank-boundary trace exchange buffers ----
// One send buffer per neighbour rank: row j = [trace_q | trace_f] of the
// local owner's side fs[j] of boundary face j, rows in boundary_face_order.
// Row-per-CTA copy: the threads of a CTA walk one contiguous row_len run, so
// loads and stores coalesce; the work is a few KB per face, HBM/latency bound.
namespace edg {
__global__ void pack_face_traces_kernel(int nsides, int row_len, int nfaces, const int32_t* __restrict__ cell,
                                        const int8_t* __restrict__ side, const double* __restrict__ tq,
                                        const double* __restrict__ tf, double* __restrict__ out) {
  // one CTA per (face, q|f) row at a time: no per-element index division
  for (int row = blockIdx.x; row < 2 * nfaces; row += gridDim.x) {
    const int j = row >> 1;
    const double* src = ((row & 1) ? tf : tq) + ((long long)__ldg(cell + j) * nsides + __ldg(side + j)) * row_len;
    double* dst = out + (long long)row * row_len;
    for (int e = threadIdx.x; e < row_len; e += blockDim.x) dst[e] = __ldg(src + e);
  }
}

__global__ void unpack_face_traces_kernel(int row_len, int nfaces, const int32_t* __restrict__ slot,
                                          const double* __restrict__ in, double* __restrict__ ghost) {
  for (int row = blockIdx.x; row < 2 * nfaces; row += gridDim.x) {
    const double* src = in + (long long)row * row_len;
    double* dst = ghost + ((long long)__ldg(slot + (row >> 1)) * 2 + (row & 1)) * row_len;
    for (int e = threadIdx.x; e < row_len; e += blockDim.x) dst[e] = __ldg(src + e);
  }
}

static unsigned copy_blocks(int rows) {
  return (unsigned)(rows < 148 * 16 ? rows : 148 * 16);   // 16 CTAs of 128 threads per SM
}

// Row gather / scatter of the sharded step (sharded.py): one warp per row of
// row_len doubles (a face trace: m * n^(d-1) = 24..125 doubles), 8 warps per CTA.
template <bool SCATTER>
__global__ void __launch_bounds__(256) rows_copy_kernel(int row_len, int nrows, const int64_t* __restrict__ idx,
                                                        const double* __restrict__ src, double* __restrict__ dst) {
  const int lane = threadIdx.x & 31;
  for (int r = blockIdx.x * 8 + (threadIdx.x >> 5); r < nrows; r += gridDim.x * 8) {
    const long long o = __ldg(idx + r) * row_len, p = (long long)r * row_len;
    const double* s = src + (SCATTER ? p : o);
    double* d = dst + (SCATTER ? o : p);
    for (int e = lane; e < row_len; e += 32) d[e] = __ldg(s + e);
  }
}
}  // namespace edg

extern "C" {

int edg_pack_face_traces(int32_t nsides, int32_t row_len, int32_t nfaces, const int32_t* cell_dev,
                         const int8_t* side_dev, const double* trace_q_dev, const double* trace_f_dev,
                         double* out_dev, void* stream) {
  if (nsides < 1 || row_len < 1 || nfaces < 0) return fail(EDG_ERR_CONFIG, "bad pack shape");
  if (nfaces == 0) return EDG_OK;
  pack_face_traces_kernel<<<copy_blocks(2 * nfaces), 128, 0, (cudaStream_t)stream>>>(
      nsides, row_len, nfaces, cell_dev, side_dev, trace_q_dev, trace_f_dev, out_dev);
  return cuda_status(check_launch());
}

int edg_gather_rows(int32_t row_len, int32_t nrows, const int64_t* idx_dev, const double* src_dev, double* dst_dev,
                    void* stream) {
  if (row_len < 1 || nrows < 0) return fail(EDG_ERR_CONFIG, "bad gather shape");
  if (nrows == 0) return EDG_OK;
  if (!idx_dev || !src_dev || !dst_dev) return fail(EDG_ERR_CONFIG, "null buffer");
  const int blocks = (nrows + 7) / 8;
  rows_copy_kernel<false><<<blocks < 148 * 8 ? blocks : 148 * 8, 256, 0, (cudaStream_t)stream>>>(row_len, nrows, idx_dev,
                                                                                              src_dev, dst_dev);
  return cuda_status(check_launch());
}

int edg_scatter_rows(int32_t row_len, int32_t nrows, const int64_t* idx_dev, const double* src_dev, double* dst_dev,
                     void* stream) {
  if (row_len < 1 || nrows < 0) return fail(EDG_ERR_CONFIG, "bad scatter shape");
  if (nrows == 0) return EDG_OK;
  if (!idx_dev || !src_dev || !dst_dev) return fail(EDG_ERR_CONFIG, "null buffer");
  const int blocks = (nrows + 7) / 8;
  rows_copy_kernel<true><<<blocks < 148 * 8 ? blocks : 148 * 8, 256, 0, (cudaStream_t)stream>>>(row_len, nrows, idx_dev,
                                                                                             src_dev, dst_dev);
  return cuda_status(check_launch());
}

int edg_unpack_face_traces(int32_t row_len, int32_t nfaces, const int32_t* slot_dev, const double* in_dev,
                           double* ghost_dev, void* stream) {
  if (row_len < 1 || nfaces < 0) return fail(EDG_ERR_CONFIG, "bad unpack shape");
  if (nfaces == 0) return EDG_OK;
  unpack_face_traces_kernel<<<copy_blocks(2 * nfaces), 128, 0, (cudaStream_t)stream>>>(row_len, nfaces, slot_dev,
                                                                                         in_dev, ghost_dev);
  return cuda_status(check_launch());
}

}  // extern "C"
