// Cell-local operators of dynamic AMR --
// replaces transfer.py:99-158:
//   * gradient_indicator / evaluate_refinement_criterion: the largest
//     |reference-space derivative| of a cell (np.max per axis, NaN-
//     propagating; the Python max over axes drops a NaN axis) and the
//     refine / keep / coarsen verdict against the hysteresis band;
//   * interpolate_volume: the parent polynomial on one of its 3^d children,
//     the per-axis interp[digit] contracted axis by axis (axis 0 first, as
//     _apply_axes, transfer.py:51-56);
//   * restrict_volume: the L2 projection of the 3^d children onto the
//     parent, sum over the children in digit order of the per-axis
//     restrict[digit] contractions.
// One CTA per cell / child / parent: these run once per mesh change, over
// the cells that change, so the kernels are written for clarity and
// coalescing (the cell block is staged in shared memory, every contraction
// pass reads it there) rather than for peak rate.
#pragma once
#include "edg_common.cuh"

namespace edg {

constexpr int kAmrThreads = 128;

// out[k][x] = sum_l T[i_ax(x)][l] in[k][x with i_ax -> l] over a staged
// (m, n^d) block, T an n x n matrix in shared memory
template <int DIM, int N>
__device__ __forceinline__ void amr_contract(const double* T, int ax, int m, const double* in, double* out) {
  constexpr int NPC = ipow(N, DIM);
  const int st = ipow(N, DIM - 1 - ax);
  for (int e = threadIdx.x; e < m * NPC; e += blockDim.x) {
    const int k = e / NPC, x = e - k * NPC;
    const int i = (x / st) % N;
    const double* src = in + k * NPC + (x - i * st);
    const double* row = T + i * N;
    double v = 0.0;
#pragma unroll
    for (int l = 0; l < N; ++l) v = fma(row[l], src[l * st], v);
    out[e] = v;
  }
}

// one CTA per cell: indicator[c], and the verdict (+1 refine, 0 keep,
// -1 coarsen; transfer.py:151-158) when verdict != null
template <int DIM, int N>
__global__ void __launch_bounds__(kAmrThreads) gradient_indicator_kernel(const double* basis, int m, int ncells,
                                                                         const double* q, const int32_t* level,
                                                                         double refine_tol, double coarsen_tol,
                                                                         int max_level, int min_level, double* ind,
                                                                         int8_t* verdict) {
  constexpr int NPC = ipow(N, DIM);
  extern __shared__ __align__(16) double smem[];
  double* sD = smem;                      // D[N][N]
  double* sQ = sD + N * N;                // (m, n^d)
  __shared__ unsigned long long sMax[DIM];
  const int c = blockIdx.x;
  for (int i = threadIdx.x; i < N * N; i += blockDim.x) sD[i] = basis[EDG_BASIS_D(N) + i];
  const double* src = q + (size_t)c * m * NPC;
  for (int i = threadIdx.x; i < m * NPC; i += blockDim.x) sQ[i] = src[i];
  if (threadIdx.x < DIM) sMax[threadIdx.x] = 0ull;
  __syncthreads();
  // per axis: NaN-propagating max of |g| over nodes and components (np.max)
  unsigned long long km[DIM];
#pragma unroll
  for (int a = 0; a < DIM; ++a) km[a] = 0ull;
  for (int e = threadIdx.x; e < m * NPC; e += blockDim.x) {
    const int k = e / NPC, x = e - k * NPC;
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
      const int st = ipow(N, DIM - 1 - a);
      const int i = (x / st) % N;
      const double* s = sQ + k * NPC + (x - i * st);
      double v = 0.0;
#pragma unroll
      for (int l = 0; l < N; ++l) v = fma(sD[i * N + l], s[l * st], v);
      const unsigned long long kv = maxkey(fabs(v));
      km[a] = kv > km[a] ? kv : km[a];
    }
  }
#pragma unroll
  for (int a = 0; a < DIM; ++a) {
    unsigned long long v = km[a];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const unsigned long long o = __shfl_xor_sync(0xffffffffu, v, off);
      v = o > v ? o : v;
    }
    if ((threadIdx.x & 31) == 0 && v) atomicMax(&sMax[a], v);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // worst = max(worst, axis max) from worst = 0.0: a NaN axis never wins
    double worst = 0.0;
#pragma unroll
    for (int a = 0; a < DIM; ++a) worst = python_max(worst, from_maxkey(sMax[a]));
    ind[c] = worst;
    if (verdict) {
      const int lv = level ? level[c] : 0;
      int8_t v = 0;
      if (worst > refine_tol && lv < max_level) v = 1;
      else if (worst < coarsen_tol && lv > min_level) v = -1;
      verdict[c] = v;
    }
  }
}

// one CTA per item: out[item] = (x)_a interp[digits[item][a]] applied to
// q[parent[item]] (parent == null: item)
template <int DIM, int N>
__global__ void __launch_bounds__(kAmrThreads) interpolate_volume_kernel(const double* basis, int m, int nitems,
                                                                         const int32_t* parent, const double* q,
                                                                         const int8_t* digits, double* out) {
  constexpr int NPC = ipow(N, DIM);
  extern __shared__ __align__(16) double smem[];
  double* sT = smem;                      // interp[3][N][N]
  double* sA = sT + 3 * N * N;
  double* sB = sA + m * NPC;
  const int it = blockIdx.x;
  const int p = parent ? parent[it] : it;
  for (int i = threadIdx.x; i < 3 * N * N; i += blockDim.x) sT[i] = basis[EDG_BASIS_INTERP(N) + i];
  const double* src = q + (size_t)p * m * NPC;
  for (int i = threadIdx.x; i < m * NPC; i += blockDim.x) sA[i] = src[i];
  __syncthreads();
  double* in = sA;
  double* o = sB;
#pragma unroll
  for (int a = 0; a < DIM; ++a) {
    amr_contract<DIM, N>(sT + digits[3 * it + a] * N * N, a, m, in, o);
    __syncthreads();
    double* t = in;
    in = o;
    o = t;
  }
  double* dst = out + (size_t)it * m * NPC;
  for (int i = threadIdx.x; i < m * NPC; i += blockDim.x) dst[i] = in[i];
}

// one CTA per parent: out[p] = sum over the 3^d children (digit order,
// row-major) of (x)_a restrict[digit_a] applied to the child
template <int DIM, int N>
__global__ void __launch_bounds__(kAmrThreads) restrict_volume_kernel(const double* basis, int m, int nparents,
                                                                      const double* children, double* out) {
  constexpr int NPC = ipow(N, DIM);
  constexpr int NCH = ipow(3, DIM);
  extern __shared__ __align__(16) double smem[];
  double* sT = smem;                      // restrict[3][N][N]
  double* sA = sT + 3 * N * N;
  double* sB = sA + m * NPC;
  double* sO = sB + m * NPC;              // running sum
  const int p = blockIdx.x;
  for (int i = threadIdx.x; i < 3 * N * N; i += blockDim.x) sT[i] = basis[EDG_BASIS_RESTR(N) + i];
  for (int ch = 0; ch < NCH; ++ch) {
    const double* src = children + ((size_t)p * NCH + ch) * m * NPC;
    __syncthreads();   // previous child done with sA / sB
    for (int i = threadIdx.x; i < m * NPC; i += blockDim.x) sA[i] = src[i];
    __syncthreads();
    double* in = sA;
    double* o = sB;
    int rest = ch;
    int dg[DIM];
#pragma unroll
    for (int a = DIM - 1; a >= 0; --a) {
      dg[a] = rest % 3;
      rest /= 3;
    }
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
      amr_contract<DIM, N>(sT + dg[a] * N * N, a, m, in, o);
      __syncthreads();
      double* t = in;
      in = o;
      o = t;
    }
    // out = part (first child), then out = out + part in child order
    for (int i = threadIdx.x; i < m * NPC; i += blockDim.x) sO[i] = ch == 0 ? in[i] : sO[i] + in[i];
  }
  __syncthreads();
  double* dst = out + (size_t)p * m * NPC;
  for (int i = threadIdx.x; i < m * NPC; i += blockDim.x) dst[i] = sO[i];
}

}  // namespace edg
