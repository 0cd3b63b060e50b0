// Shared device code of the enclavedg_b200 kernels (sm_100a, fp64).
//
// The pointwise PDE functions below evaluate exactly the operation sequence of
// the reference plugins (pde.py:27-49) and of the Euler plugin pinned in
// DESIGN.md, with the round-to-nearest intrinsics (__dmul_rn, __dadd_rn, ...)
// that nvcc never contracts into FMAs; the results are therefore bit-identical
// to numpy's on the same inputs.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/enclavedg_b200.h"

namespace edg {

constexpr int ipow(int b, int e) { return e == 0 ? 1 : b * ipow(b, e - 1); }

// Launch trace (edg_trace_next, include/enclavedg_b200.h): when a kernel is
// given a slot, thread 0 of every CTA folds the global timer at its start
// into slot[0] (atomicMin) and at its exit into slot[1] (atomicMax), so the
// slot ends up holding the launch's first-CTA start and last-CTA end in ns.
// Two atomics per CTA; a null slot costs one predicated branch.
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
struct TraceScope {
  unsigned long long* slot;
  __device__ __forceinline__ explicit TraceScope(unsigned long long* s) : slot(s) {
    if (slot && threadIdx.x == 0) atomicMin(slot, global_ns());
  }
  __device__ __forceinline__ ~TraceScope() {
    if (slot && threadIdx.x == 0) atomicMax(slot + 1, global_ns());
  }
};

struct PdeParams {
  double gamma;
  double gm1;       // gamma - 1.0, computed on the host exactly like the oracle
  double vel[3];
};

// ------------------------------------------------------------ PDE plugins --
template <int KIND, int DIM>
struct Pde;

// pde.py:27-37: F_a = a_axis * q, lambda = |a_axis|
template <int DIM>
struct Pde<EDG_PDE_ADVECTION, DIM> {
  static constexpr int M = 1;
  struct Parts {};
  __device__ __forceinline__ static Parts parts(const double*, const PdeParams&) { return {}; }
  __device__ __forceinline__ static void flux(const double* q, const Parts&, int a, const PdeParams& pp,
                                              double* f) {
    f[0] = __dmul_rn(pp.vel[a], q[0]);
  }
  __device__ __forceinline__ static double lam(const double*, const Parts&, int a, const PdeParams& pp) {
    return fabs(pp.vel[a]);
  }
  __device__ __forceinline__ static void lam_all(const double* q, const Parts& pr, const PdeParams& pp, double* l) {
#pragma unroll
    for (int a = 0; a < DIM; ++a) l[a] = lam(q, pr, a, pp);
  }
};

// pde.py:40-49: F = 0.5 * q * q (every axis), lambda = |q|
template <int DIM>
struct Pde<EDG_PDE_BURGERS, DIM> {
  static constexpr int M = 1;
  struct Parts {};
  __device__ __forceinline__ static Parts parts(const double*, const PdeParams&) { return {}; }
  __device__ __forceinline__ static void flux(const double* q, const Parts&, int, const PdeParams&,
                                              double* f) {
    f[0] = __dmul_rn(__dmul_rn(0.5, q[0]), q[0]);
  }
  __device__ __forceinline__ static double lam(const double* q, const Parts&, int, const PdeParams&) {
    return fabs(q[0]);
  }
  __device__ __forceinline__ static void lam_all(const double* q, const Parts& pr, const PdeParams& pp, double* l) {
#pragma unroll
    for (int a = 0; a < DIM; ++a) l[a] = lam(q, pr, a, pp);
  }
};

// Euler (oracle/ops.py euler):
//   inv = 1/rho; ke = (sum_i m_i*m_i) ; ke = (0.5*ke)*inv; p = gm1*(E - ke)
//   u = m_a*inv; F = (m_a, m_i*u (+p on i = a), (E + p)*u); lambda = |u| + sqrt((gamma*p)*inv)
template <int DIM>
struct Pde<EDG_PDE_EULER, DIM> {
  static constexpr int M = DIM + 2;
  struct Parts {
    double inv, p;
  };
  __device__ __forceinline__ static Parts parts(const double* q, const PdeParams& pp) {
    Parts r;
    r.inv = __drcp_rn(q[0]);
    double ke = __dmul_rn(q[1], q[1]);
#pragma unroll
    for (int i = 1; i < DIM; ++i) ke = __dadd_rn(ke, __dmul_rn(q[1 + i], q[1 + i]));
    ke = __dmul_rn(__dmul_rn(0.5, ke), r.inv);
    r.p = __dmul_rn(pp.gm1, __dsub_rn(q[1 + DIM], ke));
    return r;
  }
  // m_a without dynamic register indexing (a may be a runtime value)
  __device__ __forceinline__ static double mom(const double* q, int a) {
    double v = q[1];
#pragma unroll
    for (int i = 1; i < DIM; ++i) v = (a == i) ? q[1 + i] : v;
    return v;
  }
  __device__ __forceinline__ static void flux(const double* q, const Parts& pr, int a, const PdeParams&,
                                              double* f) {
    const double ma = mom(q, a);
    const double u = __dmul_rn(ma, pr.inv);
    f[0] = ma;
#pragma unroll
    for (int i = 0; i < DIM; ++i) {
      const double t = __dmul_rn(q[1 + i], u);
      f[1 + i] = (i == a) ? __dadd_rn(t, pr.p) : t;
    }
    f[1 + DIM] = __dmul_rn(__dadd_rn(q[1 + DIM], pr.p), u);
  }
  __device__ __forceinline__ static double lam(const double* q, const Parts& pr, int a, const PdeParams& pp) {
    const double u = __dmul_rn(mom(q, a), pr.inv);
    const double c = __dsqrt_rn(__dmul_rn(__dmul_rn(pp.gamma, pr.p), pr.inv));
    return __dadd_rn(fabs(u), c);
  }
  // every axis at once: the sound speed (one sqrt) is shared, same operations
  __device__ __forceinline__ static void lam_all(const double* q, const Parts& pr, const PdeParams& pp, double* l) {
    const double c = __dsqrt_rn(__dmul_rn(__dmul_rn(pp.gamma, pr.p), pr.inv));
#pragma unroll
    for (int a = 0; a < DIM; ++a) l[a] = __dadd_rn(fabs(__dmul_rn(q[1 + a], pr.inv)), c);
  }
};

// ------------------------------------------------- fast flux (STP only) --
// Inside the Picard iteration the result is already a non-associative fp64
// contraction (not bit-comparable with OpenBLAS), so the flux there may use a
// branch-free reciprocal (MUFU seed + two Newton steps, <= 1 ulp) and FMA
// contraction.  Riemann, corrector, FV and dt keep the exact versions above.
__device__ __forceinline__ double fast_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

template <int KIND, int DIM>
struct FastFlux {
  // all-axes flux F[a][k] of one state
  template <int M>
  __device__ __forceinline__ static void all(const double* q, const PdeParams& pp, double (&F)[DIM][M]) {
    using P = Pde<KIND, DIM>;
    const auto pr = P::parts(q, pp);
#pragma unroll
    for (int a = 0; a < DIM; ++a) P::flux(q, pr, a, pp, F[a]);
  }
};

template <int DIM>
struct FastFlux<EDG_PDE_EULER, DIM> {
  template <int M>
  __device__ __forceinline__ static void all(const double* q, const PdeParams& pp, double (&F)[DIM][M]) {
    const double inv = fast_rcp(q[0]);
    double ke = q[1] * q[1];
#pragma unroll
    for (int i = 1; i < DIM; ++i) ke = fma(q[1 + i], q[1 + i], ke);
    const double p = pp.gm1 * fma(-0.5 * ke, inv, q[1 + DIM]);
    const double ep = q[1 + DIM] + p;
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
      const double u = q[1 + a] * inv;
      F[a][0] = q[1 + a];
#pragma unroll
      for (int i = 0; i < DIM; ++i) F[a][1 + i] = (i == a) ? fma(q[1 + i], u, p) : q[1 + i] * u;
      F[a][1 + DIM] = ep * u;
    }
  }
};

// np.maximum semantics: NaN if either operand is NaN.
__device__ __forceinline__ double nan_max(double a, double b) {
  // a NaN -> a; else b NaN -> b (a > b is false); else the larger: selects, no branches
  const double m = a > b ? a : b;
  return a != a ? a : m;
}

// Rusanov outcome along +axis (kernels.py:162-173), bit-exact numpy order:
//   lam = maximum(l(lo), l(hi)); central = 0.5*(F(lo)+F(hi)); jump = 0.5*lam*(hi-lo)
template <int KIND, int DIM>
__device__ __forceinline__ void rusanov(const double* lo, const double* hi, int a, int sign,
                                        const PdeParams& pp, double* out) {
  using P = Pde<KIND, DIM>;
  constexpr int M = P::M;
  const auto pl = P::parts(lo, pp);
  const auto ph = P::parts(hi, pp);
  const double lam = nan_max(P::lam(lo, pl, a, pp), P::lam(hi, ph, a, pp));
  double fl[M], fh[M];
  P::flux(lo, pl, a, pp, fl);
  P::flux(hi, ph, a, pp, fh);
  const double hl = __dmul_rn(0.5, lam);
#pragma unroll
  for (int k = 0; k < M; ++k) {
    const double central = __dmul_rn(0.5, __dadd_rn(fl[k], fh[k]));
    const double jump = __dmul_rn(hl, __dsub_rn(hi[k], lo[k]));
    out[k] = sign >= 0 ? __dsub_rn(central, jump) : __dadd_rn(-central, jump);
  }
}

// Bit pattern ordering for non-negative doubles / NaN-propagating max.
__device__ __forceinline__ unsigned long long maxkey(double x) {
  // x >= 0 or NaN; NaN (any sign) maps above +inf.
  return (x != x) ? 0xFFFFFFFFFFFFFFFFull : (unsigned long long)__double_as_longlong(x);
}
__device__ __forceinline__ double from_maxkey(unsigned long long k) {
  return k == 0xFFFFFFFFFFFFFFFFull ? __longlong_as_double(0x7FF8000000000000ll) : __longlong_as_double((long long)k);
}

// no candidate yet: above every positive double's bits (+inf is 0x7FF0...) as
// an unsigned AND as a signed 64-bit integer, so the slots of several ranks can
// be combined with an int64 MIN all-reduce (decomposition.global_dt_slots)
constexpr unsigned long long DT_EMPTY = 0x7FFFFFFFFFFFFFFFull;

// Max of `key` over the lanes of this warp that share `seg` (segments are
// contiguous lane ranges, e.g. the nodes of one cell), then one shared-memory
// atomicMax per segment into base[seg].  All 32 lanes must call it; lanes
// without data pass key = 0.
__device__ __forceinline__ void seg_max_atomic(unsigned long long* base, int seg, unsigned long long key) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const unsigned long long v = __shfl_down_sync(0xffffffffu, key, off);
    const int sv = __shfl_down_sync(0xffffffffu, seg, off);
    if (lane + off < 32 && sv == seg && v > key) key = v;
  }
  const int prev = __shfl_up_sync(0xffffffffu, seg, 1);
  if (seg >= 0 && key != 0ull && (lane == 0 || prev != seg)) atomicMax(base + seg, key);
}

// Same contract as seg_max_atomic, but the caller passes the lane mask of its
// segment (lanes of this warp with the same `seg`): two 32-bit redux.sync
// (high word, then low word among the lanes holding the high maximum) replace
// the 5-step segmented shuffle; one shared-memory atomicMax per segment.
__device__ __forceinline__ void seg_max_redux(unsigned long long* base, int seg, unsigned mask,
                                              unsigned long long key) {
  const unsigned hi = (unsigned)(key >> 32);
  const unsigned mhi = __reduce_max_sync(mask, hi);
  const unsigned mlo = __reduce_max_sync(mask, hi == mhi ? (unsigned)key : 0u);
  const unsigned long long m = ((unsigned long long)mhi << 32) | mlo;
  if (seg >= 0 && m != 0ull && (int)(threadIdx.x & 31) == __ffs(mask) - 1) atomicMax(base + seg, m);
}

// lane mask of the lanes of this warp whose thread index lies in [lo, hi)
__device__ __forceinline__ unsigned lane_range_mask(int lo, int hi) {
  const int wb = threadIdx.x & ~31;
  const int s0 = max(lo, wb) - wb, s1 = min(hi, wb + 32) - wb;
  if (s1 <= s0) return 1u << (threadIdx.x & 31);
  const unsigned up = s1 >= 32 ? 0xffffffffu : ((1u << s1) - 1u);
  return up & ~((1u << s0) - 1u);
}

// Division by a runtime divisor d >= 1 via multiply-high (x < 2^31).
struct FastDiv {
  unsigned d, m, l;
  __device__ __forceinline__ void init(unsigned dd) {
    d = dd;
    l = 0;
    while ((1u << l) < d) ++l;
    m = l == 0 ? 0u : (unsigned)((((1ull << 32) * ((1ull << l) - d)) / d) + 1ull);
  }
  __device__ __forceinline__ unsigned div(unsigned x) const {
    if (l == 0) return x;
    const unsigned t = __umulhi(x, m);
    return (t + ((x - t) >> 1)) >> (l - 1);
  }
};

// Python-max over axes of the per-axis node maxima (kernels.py:271-273):
// lam = max(lam, ax) takes ax only if ax > lam, so a NaN axis is dropped.
__device__ __forceinline__ double python_max(double lam, double ax) { return (ax > lam) ? ax : lam; }

// candidate h / ((2p+1) * lam) (kernels.py:276-277)
__device__ __forceinline__ double dt_candidate(double h, int order, double lam) {
  return __ddiv_rn(h, __dmul_rn((double)(2 * order + 1), lam));
}

// cp.async (LDGSTS) global -> shared copies and group completion
__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(double* dst, const double* src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

// contiguous block of n doubles, all threads of the CTA cooperating
template <int THREADS>
__device__ __forceinline__ void cp_block(double* dst, const double* src, int n, int tid) {
  if (((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {
    const int n2 = n >> 1;
    for (int i = tid; i < n2; i += THREADS) cp_async16(dst + 2 * i, src + 2 * i);
    if ((n & 1) && tid == 0) cp_async8(dst + n - 1, src + n - 1);
  } else {
    for (int i = tid; i < n; i += THREADS) cp_async8(dst + i, src + i);
  }
}

// mbarrier + bulk (TMA engine) global -> shared copies
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
// expected transaction bytes without an arrival, and a plain arrival
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// L2 eviction-priority policies for streams that are read once (evict_first)
// or read again later by another CTA (evict_last), and a bulk copy that
// carries one
__device__ __forceinline__ unsigned long long l2_policy_evict_first() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ unsigned long long l2_policy_evict_last() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, unsigned bytes, unsigned long long* bar,
                                              unsigned long long policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}

inline int check_launch() {
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? EDG_OK : EDG_ERR_CUDA;
}

}  // namespace edg
