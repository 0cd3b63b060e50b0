// One compilation unit per (PDE kind, dimension): instantiates every
// PDE-specialised kernel for the supported node counts and exposes host-side
// launchers edg::unit_<name>_*.  Included by edg_k_*.cu with EDG_UNIT_KIND,
// EDG_UNIT_DIM and EDG_UNIT_NAME defined (split for parallel nvcc builds).
#include <mutex>

#include "edg_stp.cuh"
#include "edg_stp3.cuh"
#include "edg_stp2.cuh"
#include "edg_stp_ck.cuh"
#include "edg_faces.cuh"
#include "edg_corr_pipe.cuh"
#include "edg_fv.cuh"
#include "edg_dt.cuh"

#define EDG_CAT2(a, b) a##b
#define EDG_CAT(a, b) EDG_CAT2(a, b)
#define EDG_FN(suffix) EDG_CAT(EDG_CAT(unit_, EDG_UNIT_NAME), suffix)

#if EDG_UNIT_DIM == 2
#define EDG_FOR_N(X) X(2) X(3) X(4) X(5) X(6) X(7) X(8)
#else
#define EDG_FOR_N(X) X(2) X(3) X(4) X(5) X(6) X(7) X(8)
#endif

namespace edg {

// grid of a persistent kernel: SMs x resident CTAs (cached per kernel)
template <typename K>
static int persistent_grid(K kernel, int threads, size_t smem) {
  static std::mutex mu;
  static const void* keys[64];
  static int vals[64];
  static int used = 0;
  std::lock_guard<std::mutex> lock(mu);
  for (int i = 0; i < used; ++i)
    if (keys[i] == (const void*)kernel) return vals[i];
  int dev = 0, sms = 0, occ = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, smem) != cudaSuccess)
    return -1;
  const int v = sms * (occ > 0 ? occ : 1);
  if (used < 64) {
    keys[used] = (const void*)kernel;
    vals[used] = v;
    ++used;
  }
  return v;
}

template <typename K>
static int set_smem(K kernel, size_t bytes) {
  if (bytes > 48 * 1024) {
    if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) != cudaSuccess)
      return EDG_ERR_CUDA;
  }
  return EDG_OK;
}

// operator table head of order N -> this unit's constant bank (kPen).  The
// table is a pure function of N (basis.py packed_table), so it is copied once
// per process: synchronously (device to device) outside stream capture; inside
// a capture the copy becomes a node of the graph, in stream order before the
// kernel, and the next uncaptured call still makes the one-time copy.
template <int N>
static int upload_ops(const double* basis, cudaStream_t st) {
  static std::mutex mu;
  static bool done = false;
  std::lock_guard<std::mutex> lock(mu);
  if (done) return EDG_OK;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess) return EDG_ERR_CUDA;
  if (cs != cudaStreamCaptureStatusNone)
    return cudaMemcpyToSymbolAsync(kPen, basis, sizeof(double) * pen_ops(N), sizeof(double) * pen_off(N),
                                   cudaMemcpyDeviceToDevice, st) == cudaSuccess ? EDG_OK : EDG_ERR_CUDA;
  // the basis upload may still be in flight on the caller's stream
  if (cudaStreamSynchronize(st) != cudaSuccess ||
      cudaMemcpyToSymbol(kPen, basis, sizeof(double) * pen_ops(N), sizeof(double) * pen_off(N),
                         cudaMemcpyDeviceToDevice) != cudaSuccess ||
      cudaDeviceSynchronize() != cudaSuccess)
    return EDG_ERR_CUDA;
  done = true;
  return EDG_OK;
}

#ifndef EDG_STP3
#define EDG_STP3 1
#endif
// persistent-CTA launch of a predictor kernel over `blocks` work blocks with
// the launch's grid policy (StpArgs::ctas_per_sm)
template <typename K>
static int launch_stp_grid(K kern, int threads, size_t smem, int blocks, const StpArgs& a, cudaStream_t st) {
  if (set_smem(kern, smem)) return EDG_ERR_CUDA;
  int cap = persistent_grid(kern, threads, smem);
  if (cap < 0) return EDG_ERR_CUDA;
  if (a.ctas_per_sm < 0) {
    cap = blocks;
  } else if (a.ctas_per_sm > 0) {
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      return EDG_ERR_CUDA;
    if (sms * a.ctas_per_sm < cap) cap = sms * a.ctas_per_sm;
  }
  const int grid = blocks < cap ? blocks : cap;
  if (grid > 0) kern<<<grid, threads, smem, st>>>(a);
  return check_launch();
}

template <int N>
static int launch_stp_n(const StpArgs& a, cudaStream_t st) {
  constexpr int KIND = EDG_UNIT_KIND, DIM = EDG_UNIT_DIM;
  if (upload_ops<N>(a.basis, st)) return EDG_ERR_CUDA;   // constant-bank operators of order N
  if constexpr (DIM == 3 && N >= 5 && EDG_STP3) {
    // 3-D, one cell per CTA: the pencil formulation (edg_stp3.cuh)
    using C3 = Stp3Cfg<KIND, N>;
    return launch_stp_grid(stp_picard3_kernel<KIND, N>, C3::THREADS, C3::BYTES, a.nwork, a, st);
  } else if constexpr (DIM == 2 && Stp2Cfg<KIND, N>::ENABLED) {
    // 2-D Euler, n = 4: the plane formulation (edg_stp2.cuh)
    using C2 = Stp2Cfg<KIND, N>;
    return launch_stp_grid(stp_picard2_kernel<KIND, N>, C2::THREADS, C2::BYTES, (a.nwork + C2::CPB - 1) / C2::CPB, a,
                           st);
  } else {
    using Cf = StpCfg<DIM, N>;
    return launch_stp_grid(stp_picard_kernel<KIND, DIM, N>, Cf::THREADS, StpSmem<KIND, DIM, N>::BYTES,
                           (a.nwork + Cf::CPB - 1) / Cf::CPB, a, st);
  }
}

template <int N>
static int launch_stl_n(const StpArgs& a, cudaStream_t st) {
  constexpr int KIND = EDG_UNIT_KIND, DIM = EDG_UNIT_DIM;
  if constexpr (KIND != EDG_PDE_ADVECTION) {
    return EDG_ERR_NO_SPEED;   // EnclaveDgError: stp_linear requires a linear flux (kernels.py:89-90)
  } else {
    using Cf = StpCfg<DIM, N>;
    const size_t smem = sizeof(double) * (N * N + 2 * N + 1 + Cf::CPB * DIM * Pde<KIND, DIM>::M * Cf::NPC);
    auto kern = stp_linear_kernel<KIND, DIM, N>;
    if (set_smem(kern, smem)) return EDG_ERR_CUDA;
    const int blocks = (a.nwork + Cf::CPB - 1) / Cf::CPB;
    if (blocks > 0) kern<<<blocks, Cf::THREADS, smem, st>>>(a);
    return check_launch();
  }
}

int EDG_FN(_stl)(int n, const StpArgs& a, cudaStream_t st) {
  switch (n) {
#define EDG_CASE(NN) \
  case NN:           \
    return launch_stl_n<NN>(a, st);
    EDG_FOR_N(EDG_CASE)
#undef EDG_CASE
  }
  return EDG_ERR_CONFIG;
}

int EDG_FN(_stp)(int n, const StpArgs& a, cudaStream_t st) {
  switch (n) {
#define EDG_CASE(NN) \
  case NN:           \
    return launch_stp_n<NN>(a, st);
    EDG_FOR_N(EDG_CASE)
#undef EDG_CASE
  }
  return EDG_ERR_CONFIG;
}

// uniform-grid corrector: the persistent, bulk-copy double-buffered kernel
// (edg_corr_pipe.cuh); a mesh too small to give any persistent CTA a second
// group has nothing to overlap, so it gets the one-CTA-per-group kernel
template <int N>
static int launch_corr_n(bool fused, const CorrArgs& a, cudaStream_t st) {
  constexpr int KIND = EDG_UNIT_KIND, DIM = EDG_UNIT_DIM;
  if (fused && a.grid_n > 0 && a.edges_per_cell == 0) {
    using C = CorrPipe<KIND, DIM, N, true>;
    auto kern = corrector_grid_pipe_kernel<KIND, DIM, N, true>;
    if (set_smem(kern, C::BYTES)) return EDG_ERR_CUDA;
    const int grid_cap = persistent_grid(kern, C::THREADS, C::BYTES);
    if (grid_cap < 0) return EDG_ERR_CUDA;
    const int ngroups = (a.ncells - a.cell_base + C::CPB - 1) / C::CPB;
    if (ngroups > grid_cap) {
      kern<<<grid_cap, C::THREADS, C::BYTES, st>>>(a);
      return check_launch();
    }
  }
  // adaptive meshes (outcomes gathered through side_face) and small grids:
  // one CTA per group of cells (the pipelined kernel measured 25 % slower on
  // cfg5, whose 13k cells give each persistent CTA about one group)
  using Cf = CorrCfg<DIM, N>;
  const size_t smem = CorrSmem<KIND, DIM, N>::BYTES;
  const int blocks = (a.ncells - a.cell_base + Cf::CPB - 1) / Cf::CPB;
  if (blocks <= 0) return EDG_OK;
  if (fused) {
    auto kern = corrector_kernel<KIND, DIM, N, true>;
    if (set_smem(kern, smem)) return EDG_ERR_CUDA;
    kern<<<blocks, Cf::THREADS, smem, st>>>(a);
  } else {
    auto kern = corrector_kernel<KIND, DIM, N, false>;
    if (set_smem(kern, smem)) return EDG_ERR_CUDA;
    kern<<<blocks, Cf::THREADS, smem, st>>>(a);
  }
  return check_launch();
}

int EDG_FN(_corr)(int n, bool fused, const CorrArgs& a, cudaStream_t st) {
  switch (n) {
#define EDG_CASE(NN) \
  case NN:           \
    return launch_corr_n<NN>(fused, a, st);
    EDG_FOR_N(EDG_CASE)
#undef EDG_CASE
  }
  return EDG_ERR_CONFIG;
}

int EDG_FN(_faces)(int n, const FaceArgs& a, cudaStream_t st) {
  constexpr int KIND = EDG_UNIT_KIND, DIM = EDG_UNIT_DIM;
  switch (n) {
#define EDG_CASE(NN)                                                                      \
  case NN: {                                                                              \
    const long long work = (long long)a.nfaces * ipow(NN, DIM - 1);                       \
    if (work > 0) faces_rusanov_kernel<KIND, DIM, NN><<<(unsigned)((work + 127) / 128), 128, 0, st>>>(a); \
    return check_launch();                                                                \
  }
    EDG_FOR_N(EDG_CASE)
#undef EDG_CASE
  }
  return EDG_ERR_CONFIG;
}

int EDG_FN(_speed)(int order, int ncells, int npts, const double* q, const double* hmin, int h_per_cell,
                   unsigned long long* slots, const PdeParams& pp, cudaStream_t st) {
  constexpr int KIND = EDG_UNIT_KIND, DIM = EDG_UNIT_DIM;
  if (ncells > 0)
    cell_speed_kernel<KIND, DIM><<<(ncells + 7) / 8, 256, 0, st>>>(ncells, npts, q, hmin, h_per_cell, order, slots, pp);
  return check_launch();
}

int EDG_FN(_riemann)(int nfaces, int npts, const double* lo, const double* hi, int axis, int sign, double* out,
                     const PdeParams& pp, cudaStream_t st) {
  constexpr int KIND = EDG_UNIT_KIND, DIM = EDG_UNIT_DIM;
  const long long work = (long long)nfaces * npts;
  if (work > 0)
    riemann_batch_kernel<KIND, DIM><<<(unsigned)((work + 255) / 256), 256, 0, st>>>(nfaces, npts, lo, hi, axis, sign,
                                                                                  out, pp);
  return check_launch();
}

template <int K>
static int launch_fv_k(const FvArgs& a, cudaStream_t st) {
  constexpr int KIND = EDG_UNIT_KIND, DIM = EDG_UNIT_DIM;
  const size_t smem = FvSmem<KIND, DIM, K>::BYTES;
  auto kern = fv_patch_kernel<KIND, DIM, K>;
  if (set_smem(kern, smem)) return EDG_ERR_CUDA;
  if (a.npatches > a.patch_base) kern<<<a.npatches - a.patch_base, FvCfg<DIM, K>::THREADS, smem, st>>>(a);
  return check_launch();
}

int EDG_FN(_fv)(int k, const FvArgs& a, cudaStream_t st) {
  switch (k) {
    case 3:
      return launch_fv_k<3>(a, st);
    case 5:
      return launch_fv_k<5>(a, st);
    case 7:
      return launch_fv_k<7>(a, st);
    case 8:
      return launch_fv_k<8>(a, st);
  }
  return EDG_ERR_CONFIG;
}

int EDG_FN(_max_n)() {
#if EDG_UNIT_DIM == 2
  return 8;
#else
  return 8;
#endif
}

}  // namespace edg
