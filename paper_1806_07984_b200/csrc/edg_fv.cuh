// Patch finite-volume update -- replaces kernels.py:225-264.
//
// One CTA per k^d patch.  The patch and its 2d face halos (a neighbour
// patch's boundary layer, kernels.py:256-264, or the own layer at an outflow
// boundary) are staged once in shared memory as a (k+2)^d block, together
// with the state-only parts of the flux (1/rho and p for Euler).  Each thread
// owns one volume and applies, in the reference order a = 0..d-1,
//     out -= (dt / dx_a) * (F_{i+1/2} - F_{i-1/2})
// with every interface flux evaluated by the bit-exact Rusanov of
// edg_common.cuh from the ORIGINAL states (unsplit, kernels.py:240-252); an
// interface shared by two threads is evaluated twice with identical inputs,
// hence identically.  The next step's admissible-dt candidate of the patch
// (lambda over its volumes, kernels.py:267-281 with order 0) is fused into
// the epilogue.
#pragma once
#include "edg_common.cuh"

namespace edg {

struct FvArgs {
  int32_t npatches;
  const double* patch;     // [B][M][k^d]
  const int32_t* nbr;      // [B][2d] or null (halos given)
  const double* halos;     // [B][2d][M][k^(d-1)] or null
  const double* dt;
  const double* edges;     // [d] patch extent
  double* out;
  unsigned long long* dt_slots;
  double h_cell;
  uint32_t* status;
  PdeParams pp;
};

template <int DIM, int K>
struct FvCfg {
  static constexpr int NC = ipow(K, DIM);
  static constexpr int NE = ipow(K + 2, DIM);
  static constexpr int THREADS = NC >= 512 ? 512 : ((NC + 31) / 32) * 32;
};

template <int KIND, int DIM, int K>
struct FvSmem {
  static constexpr int M = Pde<KIND, DIM>::M;
  static constexpr int NPARTS = KIND == EDG_PDE_EULER ? 2 : 0;
  static constexpr size_t BYTES =
      sizeof(double) * FvCfg<DIM, K>::NE * (M + NPARTS) + sizeof(unsigned long long) * DIM;
};

// Rusanov with precomputed state parts (same arithmetic as edg::rusanov).
template <int KIND, int DIM>
__device__ __forceinline__ void rusanov_pp(const double* lo, const typename Pde<KIND, DIM>::Parts& pl,
                                           const double* hi, const typename Pde<KIND, DIM>::Parts& ph, int a,
                                           const PdeParams& pp, double* out) {
  using P = Pde<KIND, DIM>;
  constexpr int M = P::M;
  const double lam = nan_max(P::lam(lo, pl, a, pp), P::lam(hi, ph, a, pp));
  double fl[M], fh[M];
  P::flux(lo, pl, a, pp, fl);
  P::flux(hi, ph, a, pp, fh);
  const double hl = __dmul_rn(0.5, lam);
#pragma unroll
  for (int k = 0; k < M; ++k)
    out[k] = __dsub_rn(__dmul_rn(0.5, __dadd_rn(fl[k], fh[k])), __dmul_rn(hl, __dsub_rn(hi[k], lo[k])));
}

template <int KIND, int DIM, int K>
__global__ void __launch_bounds__(FvCfg<DIM, K>::THREADS) fv_patch_kernel(const FvArgs A) {
  using P = Pde<KIND, DIM>;
  using Cf = FvCfg<DIM, K>;
  constexpr int M = P::M;
  constexpr int NC = Cf::NC, NE = Cf::NE, KE = K + 2;
  constexpr int NL = ipow(K, DIM - 1);
  constexpr bool EULER = KIND == EDG_PDE_EULER;

  extern __shared__ __align__(16) double smem[];
  double* sQ = smem;                          // [M][NE]
  double* sInv = sQ + M * NE;                 // [NE] (Euler)
  double* sP = sInv + (EULER ? NE : 0);       // [NE] (Euler)
  unsigned long long* sLam = reinterpret_cast<unsigned long long*>(sQ + NE * (M + (EULER ? 2 : 0)));

  const int b = blockIdx.x;
  const int tid = threadIdx.x;
  if (tid < DIM) sLam[tid] = 0ull;
  const double* src = A.patch + (size_t)b * M * NC;

  auto ext_index = [](const int* e) {
    int idx = 0;
#pragma unroll
    for (int a = 0; a < DIM; ++a) idx = idx * KE + e[a];
    return idx;
  };
  // interior
  for (int i = tid; i < M * NC; i += blockDim.x) {
    const int k = i / NC, c = i - k * NC;
    int e[DIM], t = c;
#pragma unroll
    for (int a = DIM - 1; a >= 0; --a) {
      e[a] = t % K + 1;
      t /= K;
    }
    sQ[k * NE + ext_index(e)] = src[i];
  }
  // face halos: layer (a, s) at ext index 0 / K+1 along a
  for (int i = tid; i < 2 * DIM * M * NL; i += blockDim.x) {
    const int fs = i / (M * NL);
    const int r = i - fs * M * NL;
    const int k = r / NL, f = r - k * NL;
    const int a = fs >> 1, s = fs & 1;
    double v;
    if (A.halos) {
      v = A.halos[(size_t)b * 2 * DIM * M * NL + i];
    } else {
      const int nb = A.nbr[(size_t)b * 2 * DIM + fs];
      // neighbour below (s=0) contributes its last layer, above its first;
      // outflow (-1): own layer on that side
      const int layer = nb >= 0 ? (s == 0 ? K - 1 : 0) : (s == 0 ? 0 : K - 1);
      const int pb = nb >= 0 ? nb : b;
      int e[DIM], t = f;
      // f enumerates the non-a axes in order
#pragma unroll
      for (int ax = DIM - 1; ax >= 0; --ax) {
        if (ax == a) continue;
        e[ax] = t % K;
        t /= K;
      }
      e[a] = layer;
      int c = 0;
#pragma unroll
      for (int ax = 0; ax < DIM; ++ax) c = c * K + e[ax];
      v = A.patch[((size_t)pb * M + k) * NC + c];
    }
    int e[DIM], t = f;
#pragma unroll
    for (int ax = DIM - 1; ax >= 0; --ax) {
      if (ax == a) continue;
      e[ax] = t % K + 1;
      t /= K;
    }
    e[a] = s ? K + 1 : 0;
    sQ[k * NE + ext_index(e)] = v;
  }
  __syncthreads();
  if constexpr (EULER) {
    for (int i = tid; i < NE; i += blockDim.x) {
      double q[M];
#pragma unroll
      for (int k = 0; k < M; ++k) q[k] = sQ[k * NE + i];
      const auto pr = P::parts(q, A.pp);
      sInv[i] = pr.inv;
      sP[i] = pr.p;
    }
    __syncthreads();
  }
  const double dt = *A.dt;
  double coef[DIM];
#pragma unroll
  for (int a = 0; a < DIM; ++a) coef[a] = __ddiv_rn(dt, __ddiv_rn(A.edges[a], (double)K));

  for (int c = tid; c < NC; c += blockDim.x) {
    int e[DIM], t = c;
#pragma unroll
    for (int a = DIM - 1; a >= 0; --a) {
      e[a] = t % K + 1;
      t /= K;
    }
    const int me = ext_index(e);
    double q[M], o[M];
#pragma unroll
    for (int k = 0; k < M; ++k) o[k] = q[k] = sQ[k * NE + me];
    typename P::Parts pm{};
    if constexpr (EULER) pm = {sInv[me], sP[me]};
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
      const int st = ipow(KE, DIM - 1 - a);
      double ql[M], qh[M], fl[M], fh[M];
#pragma unroll
      for (int k = 0; k < M; ++k) {
        ql[k] = sQ[k * NE + me - st];
        qh[k] = sQ[k * NE + me + st];
      }
      typename P::Parts plo{}, phi{};
      if constexpr (EULER) {
        plo = {sInv[me - st], sP[me - st]};
        phi = {sInv[me + st], sP[me + st]};
      }
      rusanov_pp<KIND, DIM>(ql, plo, q, pm, a, A.pp, fl);
      rusanov_pp<KIND, DIM>(q, pm, qh, phi, a, A.pp, fh);
#pragma unroll
      for (int k = 0; k < M; ++k) o[k] = __dsub_rn(o[k], __dmul_rn(coef[a], __dsub_rn(fh[k], fl[k])));
    }
    bool finite = true;
#pragma unroll
    for (int k = 0; k < M; ++k) {
      A.out[((size_t)b * M + k) * NC + c] = o[k];
      finite = finite && (fabs(o[k]) <= 1.7976931348623157e308);
    }
    if (A.status && !finite) atomicAdd(A.status + 1, 1u);
    if (A.dt_slots) {
      const auto pr = P::parts(o, A.pp);
#pragma unroll
      for (int a = 0; a < DIM; ++a) atomicMax(sLam + a, maxkey(P::lam(o, pr, a, A.pp)));
    }
  }
  if (A.dt_slots) {
    __syncthreads();
    if (tid == 0) {
      double lam = 0.0;
#pragma unroll
      for (int a = 0; a < DIM; ++a) lam = python_max(lam, from_maxkey(sLam[a]));
      if (lam > 0.0)
        atomicMin(A.dt_slots + (b % EDG_DT_SLOTS),
                  (unsigned long long)__double_as_longlong(dt_candidate(A.h_cell, 0, lam)));
    }
  }
}

template <int DIM>
__global__ void boundary_layers_kernel(int m, int K, int npatches, const double* patch, double* out) {
  const int NL = DIM == 2 ? K : K * K;
  const int NC = NL * K;
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= (long long)npatches * 2 * DIM * m * NL) return;
  const int b = (int)(g / (2 * DIM * m * NL));
  const int i = (int)(g % (2 * DIM * m * NL));
  const int fs = i / (m * NL);
  const int r = i - fs * m * NL;
  const int k = r / NL, f = r - k * NL;
  const int a = fs >> 1, s = fs & 1;
  int e[DIM], t = f;
  for (int ax = DIM - 1; ax >= 0; --ax) {
    if (ax == a) continue;
    e[ax] = t % K;
    t /= K;
  }
  e[a] = s ? K - 1 : 0;
  int c = 0;
  for (int ax = 0; ax < DIM; ++ax) c = c * K + e[ax];
  out[g] = patch[((size_t)b * m + k) * NC + c];
}

}  // namespace edg
