// Patch finite-volume update -- replaces kernels.py:225-264.
//
// One CTA per k^d patch (256 threads for 8^3, two volumes per thread along
// the contiguous axis; three CTAs resident per SM).  Each thread loads the m
// components of a state (the patch volumes, then the 2d face halos: a
// neighbour patch's boundary layer, kernels.py:256-264, or the own layer at
// an outflow boundary), evaluates the state-only parts of the flux once
// (1/rho, p and the sound speed for Euler) while the values are in
// registers, and stages both in a (k+2)^d shared block whose last axis is
// padded to an odd length (conflict-free strided access).  After a single
// barrier every thread evaluates the interface fluxes of its volumes itself
// -- both neighbours of an interface evaluate it with identical inputs in the
// same (lo, hi) order, hence identically, and the interface between a
// thread's own two volumes is evaluated once -- and applies, in the
// reference order a = 0..d-1,
//     out -= (dt / dx_a) * (F_{i+1/2} - F_{i-1/2})
// from the ORIGINAL states (unsplit, kernels.py:240-252).  Every operation is
// the non-contracted round-to-nearest sequence of edg_common.cuh, so the
// result is bit-identical to the reference.  The next step's admissible-dt
// candidate of the patch (lambda over its volumes, kernels.py:267-281 with
// order 0) is fused into the epilogue.
#pragma once
#include "edg_common.cuh"

namespace edg {

struct FvArgs {
  int32_t npatches;        // end of the patch range (exclusive)
  int32_t patch_base;      // first patch of the range (0: all patches)
  const double* patch;     // [B][M][k^d]
  const int32_t* nbr;      // [B][2d] or null (halos given / grid)
  int32_t pgrid_n;         // > 0: row-major pgrid_n^d patch grid, neighbours by arithmetic
  int32_t periodic;
  const double* halos;     // [B][2d][M][k^(d-1)] or null
  const double* dt;
  const double* edges;     // [d] patch extent
  double* out;
  unsigned long long* dt_slots;
  double h_cell;
  uint32_t* status;
  PdeParams pp;
  unsigned long long* trace;   // optional launch-trace slot (TraceScope)
};

template <int DIM, int K>
struct FvCfg {
  static constexpr int NC = ipow(K, DIM);
  static constexpr int KE = K + 2;                      // extended extent (face halos)
  // EDG_FV_Z4=1 (3-D, k = 8): a thread owns volumes z and z+4 of a row and the
  // last axis is padded to 12, which makes every warp-wide state access
  // bank-conflict-free (4 lanes per row cover 4 consecutive z, rows land in
  // disjoint 4-bank-pair blocks)
#ifndef EDG_FV_Z4
#define EDG_FV_Z4 1
#endif
  static constexpr bool Z4 = EDG_FV_Z4 && DIM == 3 && K == 8;
  static constexpr int KEZ = Z4 ? 12 : ((KE % 2) ? KE : KE + 1);    // else: last axis padded to an odd length
  static constexpr int NE = ipow(KE, DIM - 1) * KEZ;    // (bank-conflict-free strided access)
  // EDG_FV_PREC=0 (default): the pressure is staged like 1/rho and c (8 arrays
  // per state).  Under Z4 the arrays are then spaced NE - 2 apart (the last two
  // padding entries of the 10 x 10 x 12 block are never addressed), which is
  // what lets three CTAs of 8 arrays share an SM: 8 * 1198 * 8 + 48 B + 1 KB
  // reserved = 77 744 B each, 233 232 of the SM's 233 472 B.  EDG_FV_PREC=1
  // recomputes the pressure from the staged state at every load (7 arrays)
#ifndef EDG_FV_PREC
#define EDG_FV_PREC 0
#endif
  static constexpr bool PREC = EDG_FV_PREC && Z4;
  static constexpr int NES = (Z4 && !PREC) ? NE - 2 : NE;   // array stride
  static constexpr int NL = ipow(K, DIM - 1);           // cells per face layer
#ifndef EDG_FV_CPT
#define EDG_FV_CPT 2
#endif
  static constexpr int CPT = (K % 2 == 0 && NC >= 256) ? EDG_FV_CPT : 1;   // volumes per thread (pairs along the last axis)
  static constexpr int THREADS = ((NC / CPT + 31) / 32) * 32;
  static constexpr int MINB = THREADS <= 256 ? 3 : 2;
};

template <int KIND, int DIM, int K>
struct FvSmem {
  static constexpr int M = Pde<KIND, DIM>::M;
  // staged parts: 1/rho, (p,) c -- with PREC the pressure is recomputed
  static constexpr int NPARTS = KIND == EDG_PDE_EULER ? (FvCfg<DIM, K>::PREC ? 2 : 3) : 0;
  static constexpr size_t BYTES = sizeof(double) * (FvCfg<DIM, K>::NES * (M + NPARTS) + DIM) +
                                  sizeof(unsigned long long) * DIM;
};

// One patch b (one CTA per patch; states read from global memory).
template <int KIND, int DIM, int K>
__device__ __forceinline__ void fv_patch_body(const FvArgs& A, const int b, double* smem) {
  using P = Pde<KIND, DIM>;
  using Cf = FvCfg<DIM, K>;
  constexpr int M = P::M;
  constexpr int NC = Cf::NC, NE = Cf::NES, NL = Cf::NL, KE = Cf::KE, KEZ = Cf::KEZ;   // NE: array stride
  constexpr int THREADS = Cf::THREADS, CPT = Cf::CPT;
  constexpr bool EULER = KIND == EDG_PDE_EULER;
  // ext strides: last axis 1, then KEZ, then KEZ*KE
  auto estride = [](int ax) { return ax == DIM - 1 ? 1 : (ax == DIM - 2 ? KEZ : KEZ * KE); };

  constexpr bool PREC = Cf::PREC;                  // pressure recomputed from the staged state
  double* sQ = smem;                               // [M][NE]
  double* sInv = sQ + M * NE;                      // [NE] (Euler)
  constexpr bool Z4 = Cf::Z4 && CPT == 2;
  double* sP = sInv + (EULER ? NE : 0);            // [NE] (Euler; not staged when PREC)
  double* sC = sP + ((EULER && !PREC) ? NE : 0);   // [NE] (Euler) sound speed
  unsigned long long* sLam = reinterpret_cast<unsigned long long*>(sC + (EULER ? NE : 0));
  double* sCoef = reinterpret_cast<double*>(sLam + DIM);   // [DIM] dt / (edge / K)

  const int tid = threadIdx.x;
  if (tid < DIM) sLam[tid] = 0ull;
  const double* src = A.patch + (size_t)b * M * NC;

  // ext index of a cell index (row-major, last axis fastest) shifted by +1
  auto ext_of_cell = [&](int c) {
    int e = 0;
#pragma unroll
    for (int a = DIM - 1; a >= 0; --a) {
      e += (c % K + 1) * estride(a);
      c /= K;
    }
    return e;
  };
  struct State {
    double q[M];
    typename P::Parts pr;
    double c;
  };
  // stage one state (m components in registers) with its parts
  auto stage = [&](int x, const double* q) {
#pragma unroll
    for (int k = 0; k < M; ++k) sQ[k * NE + x] = q[k];
    if constexpr (EULER) {
      const auto pr = P::parts(q, A.pp);
      sInv[x] = pr.inv;
      if constexpr (!PREC) sP[x] = pr.p;
      sC[x] = __dsqrt_rn(__dmul_rn(__dmul_rn(A.pp.gamma, pr.p), pr.inv));
    }
  };
  auto load = [&](int x, State& s) {
#pragma unroll
    for (int k = 0; k < M; ++k) s.q[k] = sQ[k * NE + x];
    if constexpr (EULER) {
      const double inv = sInv[x];
      double p;
      if constexpr (PREC) {
        // parts() pressure from the staged state and 1/rho (same operations)
        double ke = __dmul_rn(s.q[1], s.q[1]);
#pragma unroll
        for (int i = 1; i < DIM; ++i) ke = __dadd_rn(ke, __dmul_rn(s.q[1 + i], s.q[1 + i]));
        ke = __dmul_rn(__dmul_rn(0.5, ke), inv);
        p = __dmul_rn(A.pp.gm1, __dsub_rn(s.q[1 + DIM], ke));
      } else {
        p = sP[x];
      }
      s.pr = {inv, p};
      s.c = sC[x];
    }
  };
  // Rusanov flux along +a between lo and hi (kernels.py:162-173), exact order
  auto iface = [&](const State& lo, const State& hi, int a, double* f) {
    if constexpr (EULER) {
      const double ul = __dmul_rn(P::mom(lo.q, a), lo.pr.inv), uh = __dmul_rn(P::mom(hi.q, a), hi.pr.inv);
      const double lam = nan_max(__dadd_rn(fabs(ul), lo.c), __dadd_rn(fabs(uh), hi.c));
      double fl[M], fh[M];
      P::flux(lo.q, lo.pr, a, A.pp, fl);
      P::flux(hi.q, hi.pr, a, A.pp, fh);
      const double hl = __dmul_rn(0.5, lam);
#pragma unroll
      for (int k = 0; k < M; ++k)
        f[k] = __dsub_rn(__dmul_rn(0.5, __dadd_rn(fl[k], fh[k])), __dmul_rn(hl, __dsub_rn(hi.q[k], lo.q[k])));
    } else {
      rusanov<KIND, DIM>(lo.q, hi.q, a, 1, A.pp, f);
    }
  };

  // ---- stage interior and halo states; every global load of a thread is
  // issued before the first shared-memory store ----
  constexpr int NIT = (NC + THREADS - 1) / THREADS;
  constexpr int NHT = (2 * DIM * NL + THREADS - 1) / THREADS;
  double qi_[NIT][M], qh_[NHT][M];
  int xh_[NHT];
  // interior volume staged by (thread, u): under Z4 the volumes the thread
  // later owns (row tid / 4, z = tid % 4 and z + 4) -- a warp's stores then
  // cover 8 rows x 4 z like its state loads (conflict-free; the linear
  // assignment put rows 12 apart on overlapping banks: 4.1 wavefronts per
  // STS.64 instead of 2), and every 32-byte sector of a load is still used
  // by 4 lanes -- else tid + u * THREADS
  constexpr bool ZST = Cf::Z4 && CPT == 2 && NIT == 2;
  auto stage_cell = [&](int u) { return ZST ? (tid / (K / 2)) * K + tid % (K / 2) + u * (K / 2) : tid + u * THREADS; };
#pragma unroll
  for (int u = 0; u < NIT; ++u) {
    const int c = stage_cell(u);
#pragma unroll
    for (int k = 0; k < M; ++k) qi_[u][k] = c < NC ? __ldg(src + k * NC + c) : 0.0;
  }
#pragma unroll
  for (int u = 0; u < NHT; ++u) {
    const int i = tid + u * THREADS;
    xh_[u] = -1;
    if (i < 2 * DIM * NL) {
      const int fs = i / NL, f = i - fs * NL;
      const int a = fs >> 1, s = fs & 1;
      int e[DIM], t = f;
#pragma unroll
      for (int ax = DIM - 1; ax >= 0; --ax) {
        if (ax == a) continue;
        e[ax] = t % K;
        t /= K;
      }
      int x = 0;
#pragma unroll
      for (int ax = 0; ax < DIM; ++ax) x += (ax == a ? (s ? K + 1 : 0) : e[ax] + 1) * estride(ax);
      xh_[u] = x;
      if (A.halos) {
#pragma unroll
        for (int k = 0; k < M; ++k) qh_[u][k] = __ldg(A.halos + (((size_t)b * 2 * DIM + fs) * M + k) * NL + f);
      } else {
        int nb;
        if (A.pgrid_n > 0) {
          // Cartesian patch grid (row-major): neighbour patch by index arithmetic
          const int n = A.pgrid_n;
          int stride = 1;
          for (int ax = DIM - 1; ax > a; --ax) stride *= n;
          const int ia = (b / stride) % n;
          int j = ia + (s ? 1 : -1);
          if (j < 0 || j >= n) j = A.periodic ? (j + n) % n : -1;
          nb = j < 0 ? -1 : b + (j - ia) * stride;
        } else {
          nb = __ldg(A.nbr + (size_t)b * 2 * DIM + fs);
        }
        // neighbour below (s=0) contributes its last layer, above its first;
        // outflow (-1): own layer on that side
        e[a] = nb >= 0 ? (s == 0 ? K - 1 : 0) : (s == 0 ? 0 : K - 1);
        int c = 0;
#pragma unroll
        for (int ax = 0; ax < DIM; ++ax) c = c * K + e[ax];
        const double* ps = A.patch + (size_t)(nb >= 0 ? nb : b) * M * NC + c;
#pragma unroll
        for (int k = 0; k < M; ++k) qh_[u][k] = __ldg(ps + k * NC);
      }
    }
  }
#pragma unroll
  for (int u = 0; u < NIT; ++u)
    if (stage_cell(u) < NC) stage(ext_of_cell(stage_cell(u)), qi_[u]);
#pragma unroll
  for (int u = 0; u < NHT; ++u)
    if (xh_[u] >= 0) stage(xh_[u], qh_[u]);
  // dt / dx_a, once per CTA (kernels.py:241: dt / (h / k) with exact divisions)
  if (tid < DIM) sCoef[tid] = __ddiv_rn(*A.dt, __ddiv_rn(A.edges[tid], (double)K));
  __syncthreads();

  double o[CPT][M];
  int cv[CPT];   // own volumes
  {
  // ---- own volumes (CPT consecutive along the last axis) ----
  // volumes c0 + j * DZ: consecutive pairs, or (Z4) z and z + k/2
  constexpr int DZ = Z4 ? K / 2 : 1;
  const int c0 = Z4 ? (tid / (K / 2)) * K + tid % (K / 2) : tid * CPT;
  const int x0 = c0 < NC ? ext_of_cell(c0) : ext_of_cell(0);
#pragma unroll
  for (int j = 0; j < CPT; ++j) cv[j] = c0 + j * DZ;
  // EDG_FV_JOUTER=1 (with Z4): volume-outer loop order -- one volume's state,
  // both interface fluxes and its update are live at a time (the axis-outer
  // order keeps both volumes' states live: spills at the 3-CTA register cap)
#ifndef EDG_FV_JOUTER
#define EDG_FV_JOUTER 1
#endif
  if constexpr (Z4 && EDG_FV_JOUTER) {
#pragma unroll
    for (int j = 0; j < CPT; ++j) {
      State mj;
      load(x0 + j * DZ, mj);
#pragma unroll
      for (int k = 0; k < M; ++k) o[j][k] = mj.q[k];
#pragma unroll
      for (int a = 0; a < DIM; ++a) {
        const double coef = sCoef[a];
        const int st = estride(a);
        State nb;
        double fl[M], fh[M];
        load(x0 + j * DZ - st, nb);
        iface(nb, mj, a, fl);
        load(x0 + j * DZ + st, nb);
        iface(mj, nb, a, fh);
#pragma unroll
        for (int k = 0; k < M; ++k) o[j][k] = __dsub_rn(o[j][k], __dmul_rn(coef, __dsub_rn(fh[k], fl[k])));
      }
    }
  } else {
  State me[CPT];
#pragma unroll
  for (int j = 0; j < CPT; ++j) {
    load(x0 + j * DZ, me[j]);
#pragma unroll
    for (int k = 0; k < M; ++k) o[j][k] = me[j].q[k];
  }
#pragma unroll
  for (int a = 0; a < DIM; ++a) {
    const double coef = sCoef[a];
    const int st = estride(a);
    if (a == DIM - 1 && CPT == 2 && !Z4) {
      // interfaces (x0-1 | x0), (x0 | x0+1) shared, (x0+1 | x0+2)
      State nb;
      double fL[M], fM[M], fU[M];
      load(x0 - 1, nb);
      iface(nb, me[0], a, fL);
      iface(me[0], me[1], a, fM);
      load(x0 + 2, nb);
      iface(me[1], nb, a, fU);
#pragma unroll
      for (int k = 0; k < M; ++k) {
        o[0][k] = __dsub_rn(o[0][k], __dmul_rn(coef, __dsub_rn(fM[k], fL[k])));
        o[1][k] = __dsub_rn(o[1][k], __dmul_rn(coef, __dsub_rn(fU[k], fM[k])));
      }
    } else {
#pragma unroll
      for (int j = 0; j < CPT; ++j) {
        State nb;
        double fl[M], fh[M];
        load(x0 + j * DZ - st, nb);
        iface(nb, me[j], a, fl);
        load(x0 + j * DZ + st, nb);
        iface(me[j], nb, a, fh);
#pragma unroll
        for (int k = 0; k < M; ++k) o[j][k] = __dsub_rn(o[j][k], __dmul_rn(coef, __dsub_rn(fh[k], fl[k])));
      }
    }
  }
  }

  }  // volume-owner variant

  // ---- write back, non-finite count, next-step dt candidate ----
  // The patch is the dt unit (admissible_dt with order 0 over its volumes):
  // per axis a NaN-propagating max over the volumes, then the python max over
  // the axes (NaN axes dropped, kernels.py:267-281).  NaN axes are flagged in
  // shared memory first; then one NaN-free maximum over volumes and the
  // remaining axes is reduced (one warp butterfly, one shared atomic per warp).
  unsigned* const nanbits = reinterpret_cast<unsigned*>(sLam + 1);
  double lv[CPT][DIM];
#pragma unroll
  for (int j = 0; j < CPT; ++j) {
    const int c = cv[j];
    if (c < NC) {
      bool finite = true;
#pragma unroll
      for (int k = 0; k < M; ++k) {
        A.out[((size_t)b * M + k) * NC + c] = o[j][k];
        finite = finite && (fabs(o[j][k]) <= 1.7976931348623157e308);
      }
      if (A.status && !finite) atomicAdd(A.status + 1, 1u);
      if (A.dt_slots) {
        const auto pr = P::parts(o[j], A.pp);
        P::lam_all(o[j], pr, A.pp, lv[j]);
#pragma unroll
        for (int a = 0; a < DIM; ++a)
          if (lv[j][a] != lv[j][a]) atomicOr(nanbits, 1u << a);
      }
    }
  }
  if (A.dt_slots) {
    __syncthreads();
    const unsigned nb = *nanbits;
    double lmax = 0.0;
#pragma unroll
    for (int j = 0; j < CPT; ++j)
      if (cv[j] < NC) {
#pragma unroll
        for (int a = 0; a < DIM; ++a)
          if (!((nb >> a) & 1u)) lmax = lv[j][a] > lmax ? lv[j][a] : lmax;
      }
    unsigned long long key = (unsigned long long)__double_as_longlong(lmax);   // >= 0, NaN-free
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const unsigned long long v = __shfl_xor_sync(0xffffffffu, key, off);
      key = v > key ? v : key;
    }
    if ((tid & 31) == 0 && key) atomicMax(sLam, key);
    __syncthreads();
    if (tid == 0) {
      const double lam = __longlong_as_double((long long)*sLam);
      if (lam > 0.0)
        atomicMin(A.dt_slots + (b % EDG_DT_SLOTS),
                  (unsigned long long)__double_as_longlong(dt_candidate(A.h_cell, 0, lam)));
    }
  }
}

template <int KIND, int DIM, int K, int MINB = FvCfg<DIM, K>::MINB>
__global__ void __launch_bounds__(FvCfg<DIM, K>::THREADS, MINB) fv_patch_kernel(const FvArgs A) {
  const TraceScope trace_scope(A.trace);
  extern __shared__ __align__(16) double smem[];
  fv_patch_body<KIND, DIM, K>(A, A.patch_base + (int)blockIdx.x, smem);
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
