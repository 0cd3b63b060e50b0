// Admissible-timestep reduction -- replaces kernels.py:267-281.
//
// One warp per cell (or FV patch): lanes stride over the nodes, keep the
// per-axis maximum wave speed as a NaN-propagating 64-bit key (numpy .max()
// semantics), reduce it with warp shuffles, and lane 0 applies the Python
// max over axes (a NaN axis is dropped, kernels.py:271-273), skips lam <= 0
// (kernels.py:274-275) and forms h / ((2p+1) lam).  The CTA minimum goes to
// one of EDG_DT_SLOTS slots with a 64-bit atomicMin on the bit pattern
// (positive doubles order like their bits), and edg_dt_finalize folds the
// slots into dt = cfl * min (kernels.py:281) on the device, so a whole
// time step can be captured in a CUDA graph without a host round trip.
#pragma once
#include "edg_common.cuh"

namespace edg {

template <int KIND, int DIM>
__global__ void __launch_bounds__(256) cell_speed_kernel(int ncells, int npts, const double* q,
                                                         const double* hmin, int h_per_cell, int order,
                                                         unsigned long long* slots, PdeParams pp) {
  using P = Pde<KIND, DIM>;
  constexpr int M = P::M;
  __shared__ unsigned long long sBest[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x * 8 + warp;
  unsigned long long best = DT_EMPTY;
  if (c < ncells) {
    unsigned long long key[DIM];
#pragma unroll
    for (int a = 0; a < DIM; ++a) key[a] = 0ull;
    const double* qc = q + (size_t)c * M * npts;
    for (int i = lane; i < npts; i += 32) {
      double s[M];
#pragma unroll
      for (int k = 0; k < M; ++k) s[k] = qc[(size_t)k * npts + i];
      const auto pr = P::parts(s, pp);
      double l[DIM];
      P::lam_all(s, pr, pp, l);
#pragma unroll
      for (int a = 0; a < DIM; ++a) {
        const unsigned long long kk = maxkey(l[a]);
        key[a] = kk > key[a] ? kk : key[a];
      }
    }
#pragma unroll
    for (int a = 0; a < DIM; ++a)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long v = __shfl_xor_sync(0xffffffffu, key[a], o);
        key[a] = v > key[a] ? v : key[a];
      }
    if (lane == 0) {
      double lam = 0.0;
#pragma unroll
      for (int a = 0; a < DIM; ++a) lam = python_max(lam, from_maxkey(key[a]));
      if (lam > 0.0)
        best = (unsigned long long)__double_as_longlong(dt_candidate(hmin[h_per_cell ? c : 0], order, lam));
    }
  }
  if (lane == 0) sBest[warp] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long b = DT_EMPTY;
    for (int i = 0; i < 8; ++i) b = sBest[i] < b ? sBest[i] : b;
    if (b != DT_EMPTY) atomicMin(slots + (blockIdx.x % EDG_DT_SLOTS), b);
  }
}

static __global__ void dt_slots_reset_kernel(unsigned long long* slots) {
  for (int i = threadIdx.x; i < EDG_DT_SLOTS; i += blockDim.x) slots[i] = DT_EMPTY;
}

static __global__ void dt_finalize_kernel(unsigned long long* slots, double cfl, double* dt, double* hist, int step,
                                   uint32_t* status, unsigned long long* trace) {
  const TraceScope trace_scope(trace);
  __shared__ unsigned long long s[EDG_DT_SLOTS];
  const int t = threadIdx.x;
  s[t] = slots[t];
  slots[t] = DT_EMPTY;
  __syncthreads();
  for (int o = EDG_DT_SLOTS / 2; o > 0; o >>= 1) {
    if (t < o) s[t] = s[t + o] < s[t] ? s[t + o] : s[t];
    __syncthreads();
  }
  if (t == 0) {
    double v;
    if (s[0] == DT_EMPTY) {
      v = __longlong_as_double(0x7FF8000000000000ll);
      if (status) atomicOr(status, 1u);
    } else {
      v = __dmul_rn(cfl, __longlong_as_double((long long)s[0]));
    }
    *dt = v;
    // status[3]: 1-based index of the first step whose result was non-finite
    if (status && status[1] != 0u && status[3] == 0u) status[3] = status[2];
    if (hist) {
      // step >= 0: explicit slot; step < 0: device counter status[2] with
      // capacity -step (graph-replay friendly)
      if (step >= 0) {
        hist[step] = v;
      } else if (status) {
        const unsigned idx = status[2]++;
        if (idx < (unsigned)(-step)) hist[idx] = v;
      }
    }
  }
}

// ---------------------------------------- Picard-count ordering of cells --
// Counting sort of the cells by their last Picard iteration count, so that a
// CTA of the next predictor launch holds cells that will iterate alike (the
// CTA runs until its slowest cell converges).  Order inside a bucket is not
// deterministic; results are, because cells are independent.
constexpr int ORDER_BINS = 64;

static __global__ void order_hist_kernel(int n, const int32_t* its, int32_t* hist) {
  __shared__ int32_t h[ORDER_BINS];
  for (int i = threadIdx.x; i < ORDER_BINS; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < n) atomicAdd(&h[min(max(its[c], 0), ORDER_BINS - 1)], 1);
  __syncthreads();
  for (int i = threadIdx.x; i < ORDER_BINS; i += blockDim.x)
    if (h[i]) atomicAdd(&hist[i], h[i]);
}

static __global__ void order_scan_kernel(int32_t* hist, int32_t* offs) {
  // descending iteration count first (the heaviest CTAs start earliest):
  // exclusive prefix sum over the bins in descending order, one warp, two
  // bins per lane (a serial loop here cost ~20 us of dependent L2 loads)
  static_assert(ORDER_BINS == 64, "one warp, two bins per lane");
  const int lane = threadIdx.x;
  const int b0 = ORDER_BINS - 1 - 2 * lane, b1 = b0 - 1;
  const int h0 = hist[b0], h1 = hist[b1];
  int s = h0 + h1;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, s, off);
    if (lane >= off) s += v;
  }
  const int excl = s - h0 - h1;
  offs[b0] = excl;
  offs[b1] = excl + h0;
  hist[b0] = 0;
  hist[b1] = 0;
}

static __global__ void order_scatter_kernel(int n, const int32_t* its, int32_t* offs, int32_t* order) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const bool ok = c < n;
  const int b = ok ? min(max(its[c], 0), ORDER_BINS - 1) : -1;
  // warp-aggregated slot reservation per bucket
  const unsigned peers = __match_any_sync(0xffffffffu, b);
  const int leader = __ffs(peers) - 1;
  const int lane = threadIdx.x & 31;
  int base = 0;
  if (ok && lane == leader) base = atomicAdd(&offs[b], __popc(peers));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (ok) order[base + __popc(peers & ((1u << lane) - 1u))] = c;
}

template <int KIND, int DIM>
__global__ void riemann_batch_kernel(int nfaces, int npts, const double* lo, const double* hi, int axis, int sign,
                                     double* out, PdeParams pp) {
  constexpr int M = Pde<KIND, DIM>::M;
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= (long long)nfaces * npts) return;
  const int f = (int)(g / npts), i = (int)(g % npts);
  double l[M], h[M], o[M];
#pragma unroll
  for (int k = 0; k < M; ++k) {
    l[k] = lo[((size_t)f * M + k) * npts + i];
    h[k] = hi[((size_t)f * M + k) * npts + i];
  }
  rusanov<KIND, DIM>(l, h, axis, sign, pp, o);
#pragma unroll
  for (int k = 0; k < M; ++k) out[((size_t)f * M + k) * npts + i] = o[k];
}

}  // namespace edg
