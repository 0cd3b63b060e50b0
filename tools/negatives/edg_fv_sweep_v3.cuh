// Patch finite-volume update, plane-sweep formulation for 3-D Euler 8^3
// patches (config 4) -- replaces kernels.py:225-264 on that shape; every other
// (pde, dim, k) keeps fv_patch_kernel (edg_fv.cuh).
//
// The volume-owner kernel evaluates each interior interface twice (by both
// neighbours) and is bound by FP64 issue (ncu: FP64 pipe 60 % at 27 % of HBM).
// Here every interface flux is evaluated ONCE:
//   * one CTA per patch, 96 threads: 64 column threads (y, z) that march along
//     axis 0 (x = -1 .. 8, the two end planes are the x halos) and 32 halo
//     threads that own the y / z halo states of the current plane;
//   * a column thread keeps the previous and the current state of its column
//     in registers (with 1/rho, p, c evaluated once per state), so the axis-0
//     interface (x - 1/2) needs no shared memory at all, and F_0 and the wave
//     speed of the current state are reused for the next interface;
//   * per plane the 96 states are published to shared memory; column threads
//     evaluate their upper y and z interfaces (towards interior neighbours),
//     halo threads the 32 interfaces between a halo state and its interior
//     neighbour, all into a per-plane flux buffer; after a barrier each column
//     thread reads the two lower / two upper fluxes of its volume.
// The update keeps the reference order (kernels.py:240-252)
//     out = ((q - c0 (Fx+ - Fx-)) - c1 (Fy+ - Fy-)) - c2 (Fz+ - Fz-)
// with non-contracted round-to-nearest operations from the ORIGINAL states,
// so the result is bit-identical to fv_patch_kernel and to the reference.
// Volume x of a column is finished when the interface (x + 1/2) is known (one
// plane later); the patch's admissible-dt candidate of the NEW state
// (kernels.py:267-281, order 0) is folded in as the volumes are finished.
#pragma once
#include "edg_fv.cuh"

namespace edg {

#ifndef EDG_FV_SWEEP
#define EDG_FV_SWEEP 1
#endif
#ifndef EDG_FV_SWEEP_MINB
#define EDG_FV_SWEEP_MINB 2
#endif
// planes in flight (cp.async) ahead of the plane being consumed
#ifndef EDG_FV_SWEEP_D
#define EDG_FV_SWEEP_D 6
#endif

template <int KIND, int DIM, int K>
struct FvSweep {
  static constexpr bool ENABLED = EDG_FV_SWEEP && KIND == EDG_PDE_EULER && DIM == 3 && K == 8;
  static constexpr int COLS = K * K;          // threads per role: columns (warps 0-1), finishers (2-3), y (4-5), z (6-7)
  static constexpr int HALO = 4 * K;          // halo threads (warp 8): y+, y-, z+, z- rows of the plane
  static constexpr int THREADS = 4 * COLS + HALO;
  static constexpr int NV = 8;                // q[5], 1/rho, p, c
  static constexpr int SP = COLS + HALO;      // states of one plane
  static constexpr int NIF = (K + 1) * K;     // interfaces of one transverse axis per plane
  static constexpr int D = EDG_FV_SWEEP_D < K + 2 ? EDG_FV_SWEEP_D : K + 2;
  static constexpr int R = D + 2;             // ring slots: plane p - 1 (re-read), p, and D in flight
  static constexpr int M = KIND == EDG_PDE_EULER ? DIM + 2 : 1;
  static constexpr size_t BYTES =
      sizeof(double) * (R * M * SP + 2 * NV * SP + 4 * M * NIF + 2 * M * COLS + 2 * (M + 1) * COLS + 2 * M * COLS);
};

template <int K, int MINB>
__global__ void __launch_bounds__(FvSweep<EDG_PDE_EULER, 3, K>::THREADS, MINB) fv_sweep_kernel(const FvArgs A) {
  const TraceScope trace_scope(A.trace);
  constexpr int KIND = EDG_PDE_EULER, DIM = 3;
  using P = Pde<KIND, DIM>;
  using Cf = FvSweep<KIND, DIM, K>;
  constexpr int M = P::M, NC = K * K * K, NL = K * K;
  constexpr int COLS = Cf::COLS, NV = Cf::NV, NIF = Cf::NIF, SP = Cf::SP;
  constexpr int H_YP = COLS, H_ZP = COLS + 2 * K;   // halo rows: y+, y-, z+, z-

  constexpr int D = Cf::D, R = Cf::R;
  extern __shared__ __align__(16) double smem[];
  typedef double (*RingT)[M][SP];
  typedef double (*StT)[NV][SP];
  typedef double (*FlT)[M][NIF];
  typedef double (*ColT)[M][COLS];
  typedef double (*ColXT)[M + 1][COLS];
  RingT sR = reinterpret_cast<RingT>(smem);                      // [R] raw states of the planes in flight
  StT sS = reinterpret_cast<StT>(smem + R * M * SP);             // [2] states (+ parts) of planes v, by parity of v
  FlT sFY = reinterpret_cast<FlT>(&sS[2][0][0]);                 // [2] y interfaces j = 0..K of plane v: [j * K + z]
  FlT sFZ = reinterpret_cast<FlT>(&sFY[2][0][0]);                // [2] z interfaces: [y * (K + 1) + j]
  ColT sO1 = reinterpret_cast<ColT>(&sFZ[2][0][0]);              // [2] q - c0 (Fx+ - Fx-) of the volumes of plane v
  ColXT sX = reinterpret_cast<ColXT>(&sO1[2][0][0]);             // [2] F_0 and wave speed of plane v (thread-private)
  ColT sFX = reinterpret_cast<ColT>(&sX[2][0][0]);               // [2] x interface v - 1/2 (thread-private)
  __shared__ double sCoef[DIM];
  __shared__ unsigned long long sLam;
  __shared__ unsigned sNan;

  const int tid = threadIdx.x;
  const int b = A.patch_base + (int)blockIdx.x;
  const int role = tid / COLS;          // 0 C (columns), 1 F (finishers), 2 Y, 3 Z, 4 H (warp-uniform)
  const int lt = tid - role * COLS;     // index within the role
  if (tid == 0) {
    sLam = 0ull;
    sNan = 0u;
  }
  // dt / dx_a, once per CTA (kernels.py:241: dt / (h / k) with exact divisions)
  if (tid < DIM) sCoef[tid] = __ddiv_rn(*A.dt, __ddiv_rn(A.edges[tid], (double)K));

  struct State {
    double q[M];
    double inv, p, c;
  };
  auto eval_parts = [&](State& s) {
    const auto pr = P::parts(s.q, A.pp);
    s.inv = pr.inv;
    s.p = pr.p;
    s.c = __dsqrt_rn(__dmul_rn(__dmul_rn(A.pp.gamma, pr.p), pr.inv));
  };
  auto publish = [&](int par, int x, const State& s) {
#pragma unroll
    for (int k = 0; k < M; ++k) sS[par][k][x] = s.q[k];
    sS[par][M][x] = s.inv;
    sS[par][M + 1][x] = s.p;
    sS[par][M + 2][x] = s.c;
  };
  auto fetch = [&](int par, int x, State& s) {
#pragma unroll
    for (int k = 0; k < M; ++k) s.q[k] = sS[par][k][x];
    s.inv = sS[par][M][x];
    s.p = sS[par][M + 1][x];
    s.c = sS[par][M + 2][x];
  };
  // F_a(s) and |u_a| + c
  auto flux_of = [&](const State& s, int a, double* f, double& l) {
    const typename P::Parts pr{s.inv, s.p};
    P::flux(s.q, pr, a, A.pp, f);
    l = __dadd_rn(fabs(__dmul_rn(P::mom(s.q, a), s.inv)), s.c);
  };
  // Rusanov flux between lo and hi (kernels.py:162-173), exact order; the
  // wave-speed maximum propagates NaN like nan_max (lo's first), branch-free
  auto combine = [&](const double* qlo, const double* fl, double ll, const double* qhi, const double* fh, double lh,
                     double* f) {
    double lam = ll > lh ? ll : lh;      // lh NaN -> lh
    lam = ll != ll ? ll : lam;
    const double hl = __dmul_rn(0.5, lam);
#pragma unroll
    for (int k = 0; k < M; ++k)
      f[k] = __dsub_rn(__dmul_rn(0.5, __dadd_rn(fl[k], fh[k])), __dmul_rn(hl, __dsub_rn(qhi[k], qlo[k])));
  };
  auto neighbour = [&](int a, int s) -> int {
    if (A.pgrid_n > 0) {
      const int n = A.pgrid_n;
      int stride = 1;
      for (int ax = DIM - 1; ax > a; --ax) stride *= n;
      const int ia = (b / stride) % n;
      int j = ia + (s ? 1 : -1);
      if (j < 0 || j >= n) j = A.periodic ? (j + n) % n : -1;
      return j < 0 ? -1 : b + (j - ia) * stride;
    }
    return __ldg(A.nbr + (size_t)b * 2 * DIM + 2 * a + s);
  };

  // ---- per-thread source pointers and slots ----
  // C: own planes and the x-/x+ halo planes (component strides cs_m / cs_p);
  // H: its halo state of plane x at hp + x * hxs (component stride hcs)
  const double* own = A.patch + (size_t)b * M * NC + lt;
  const double *pm = own, *pp_ = own, *hp = own;
  int cs_m = NC, cs_p = NC, hcs = NC, hxs = NL;
  int i_lo = 0, i_hi = 0, i_slot = 0;   // Y / Z / H: state rows of the interface and its flux slot
  int h_axis = 1, h_hi = 0, h_row = H_YP;
  bool work = true;                     // Y / Z: the thread owns an interior interface
  const int cy = lt / K, cz = lt - cy * K;
  if (role == 0) {
    if (A.halos) {
      pm = A.halos + ((size_t)b * 2 * DIM + 0) * M * NL + lt;
      pp_ = A.halos + ((size_t)b * 2 * DIM + 1) * M * NL + lt;
      cs_m = cs_p = NL;
    } else {
      // neighbour below contributes its last plane, above its first;
      // outflow (-1): own plane on that side (kernels.py:256-264)
      const int nm = neighbour(0, 0), np = neighbour(0, 1);
      pm = A.patch + (size_t)(nm >= 0 ? nm : b) * M * NC + (nm >= 0 ? (K - 1) * NL : 0) + lt;
      pp_ = A.patch + (size_t)(np >= 0 ? np : b) * M * NC + (np >= 0 ? 0 : (K - 1) * NL) + lt;
    }
  } else if (role == 2) {
    // interface j = 1 + lt / K between rows j - 1 and j at z = lt % K
    work = lt < (K - 1) * K;
    i_lo = work ? lt : 0;
    i_hi = i_lo + K;
    i_slot = i_lo + K;
  } else if (role == 3) {
    // interface j = 1 + lt % (K - 1) of row y = lt / (K - 1)
    work = lt < (K - 1) * K;
    const int yy = work ? lt / (K - 1) : 0, j = work ? 1 + lt - yy * (K - 1) : 1;
    i_lo = yy * K + j - 1;
    i_hi = i_lo + 1;
    i_slot = yy * (K + 1) + j;
  } else if (role == 4) {
    const int side = lt / K, t = lt - side * K;                 // side: 0 y+, 1 y-, 2 z+, 3 z-
    h_axis = 1 + (side >> 1);
    h_hi = (side & 1) ^ 1;                                      // 1: the halo state is the upper one
    h_row = COLS + side * K + t;
    const int e_in = h_hi ? K - 1 : 0;                          // interior neighbour's coordinate on the axis
    i_lo = h_axis == 1 ? e_in * K + t : t * K + e_in;           // interior row
    i_slot = h_axis == 1 ? (h_hi ? K : 0) * K + t : t * (K + 1) + (h_hi ? K : 0);
    const int fs = 2 * h_axis + h_hi;
    if (A.halos) {
      hp = A.halos + ((size_t)b * 2 * DIM + fs) * M * NL + t;
      hcs = NL;
      hxs = K;
    } else {
      const int nb = neighbour(h_axis, h_hi);
      const int e = nb >= 0 ? (h_hi ? 0 : K - 1) : (h_hi ? K - 1 : 0);
      hp = A.patch + (size_t)(nb >= 0 ? nb : b) * M * NC + (h_axis == 1 ? e * K + t : t * K + e);
    }
  }

  double lv[DIM] = {0.0, 0.0, 0.0};
  unsigned nanmask = 0u;
  // item n of the ring: C plane n - 1 (x = -1 .. K), H plane n (0 .. K-1);
  // every thread copies (and later reads) only its own element
  auto issue = [&](int n) {
    if (role == 0 && n <= K + 1) {
      const int x = n - 1;
      const double* src = x < 0 ? pm : (x < K ? own + x * NL : pp_);
      const int cs = x < 0 ? cs_m : (x < K ? NC : cs_p);
#pragma unroll
      for (int k = 0; k < M; ++k) cp_async8(&sR[n % R][k][lt], src + (size_t)k * cs);
    } else if (role == 4 && n < K) {
#pragma unroll
      for (int k = 0; k < M; ++k) cp_async8(&sR[n % R][k][COLS + lt], hp + (size_t)n * hxs + (size_t)k * hcs);
    }
    cp_async_commit();
  };
#pragma unroll
  for (int n = 0; n < D; ++n) issue(n);
  __syncthreads();                      // sCoef, sLam, sNan

  // ---- phases p = -1 .. K+1, one barrier each; no role keeps state in
  // registers across a phase ----
  //  C: plane p (prv = plane p - 1): parts, F_0, the interface p - 1/2,
  //     q - c0 (Fx+ - Fx-) of volume p - 1, the state of plane p published
  //  Y, Z, H: the y / z interfaces of plane p - 1; H also publishes the halo
  //     states of plane p
  //  F: volume p - 2 finished from the x part and the y / z fluxes of plane p - 2
#pragma unroll 1
  for (int p = -1; p <= K + 1; ++p) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(D - 1) : "memory");   // item p + 1 has landed
    const int par = p & 1, ppar = par ^ 1;
    if (role == 0) {
      if (p <= K) {
        const int n = p + 1;
        State s;
        double f0[M], l0;
#pragma unroll
        for (int k = 0; k < M; ++k) s.q[k] = sR[n % R][k][lt];
        eval_parts(s);
        flux_of(s, 0, f0, l0);
        if (p >= 0) {
          double qv[M], fv[M], fx[M];
#pragma unroll
          for (int k = 0; k < M; ++k) {
            qv[k] = sR[(n - 1) % R][k][lt];
            fv[k] = sX[ppar][k][lt];
          }
          combine(qv, fv, sX[ppar][M][lt], s.q, f0, l0, fx);   // interface p - 1/2
          if (p >= 1) {
            const double c0 = sCoef[0];
#pragma unroll
            for (int k = 0; k < M; ++k)
              sO1[ppar][k][lt] = __dsub_rn(qv[k], __dmul_rn(c0, __dsub_rn(fx[k], sFX[ppar][k][lt])));
          }
#pragma unroll
          for (int k = 0; k < M; ++k) sFX[par][k][lt] = fx[k];
        }
        if (p < K) {
#pragma unroll
          for (int k = 0; k < M; ++k) sX[par][k][lt] = f0[k];
          sX[par][M][lt] = l0;
          if (p >= 0) publish(par, lt, s);
        }
      }
    } else if (role == 1) {
      if (p >= 2) {
        // volume v = p - 2 of this column is complete
        const int v = p - 2;
        const double c1 = sCoef[1], c2 = sCoef[2];
        double o[M];
        bool finite = true;
        double* dst = A.out + (size_t)b * M * NC + v * NL + lt;
#pragma unroll
        for (int k = 0; k < M; ++k) {
          const double dy = __dmul_rn(c1, __dsub_rn(sFY[par][k][lt + K], sFY[par][k][lt]));
          const double dz = __dmul_rn(c2, __dsub_rn(sFZ[par][k][cy * (K + 1) + cz + 1], sFZ[par][k][cy * (K + 1) + cz]));
          o[k] = __dsub_rn(__dsub_rn(sO1[par][k][lt], dy), dz);
          dst[(size_t)k * NC] = o[k];
          finite = finite && (fabs(o[k]) <= 1.7976931348623157e308);
        }
        if (A.status && !finite) atomicAdd(A.status + 1, 1u);
        if (A.dt_slots) {
          const auto pr = P::parts(o, A.pp);
          double l[DIM];
          P::lam_all(o, pr, A.pp, l);
#pragma unroll
          for (int a = 0; a < DIM; ++a) {
            if (l[a] != l[a]) nanmask |= 1u << a;
            else lv[a] = l[a] > lv[a] ? l[a] : lv[a];
          }
        }
      }
    } else if (role == 4) {
      if (p >= 1 && p <= K) {
        // boundary interface of plane p - 1: halo state | interior state (both published last phase)
        State in, hs;
        double fa[M], la, fb[M], lb, f[M];
        fetch(ppar, i_lo, in);
        fetch(ppar, h_row, hs);
        flux_of(in, h_axis, fa, la);
        flux_of(hs, h_axis, fb, lb);
        if (h_hi) combine(in.q, fa, la, hs.q, fb, lb, f);
        else combine(hs.q, fb, lb, in.q, fa, la, f);
        double* dstf = h_axis == 1 ? &sFY[ppar][0][i_slot] : &sFZ[ppar][0][i_slot];
#pragma unroll
        for (int k = 0; k < M; ++k) dstf[k * NIF] = f[k];
      }
      if (p >= 0 && p < K) {
        State hs;
#pragma unroll
        for (int k = 0; k < M; ++k) hs.q[k] = sR[p % R][k][COLS + lt];
        eval_parts(hs);
        publish(par, h_row, hs);
      }
    } else if (p >= 1 && p <= K && work) {
      // interior interface of plane p - 1 along y (role 2) / z (role 3)
      State lo, hi;
      double fl[M], ll, fh[M], lh, f[M];
      fetch(ppar, i_lo, lo);
      fetch(ppar, i_hi, hi);
      if (role == 2) {
        flux_of(lo, 1, fl, ll);
        flux_of(hi, 1, fh, lh);
      } else {
        flux_of(lo, 2, fl, ll);
        flux_of(hi, 2, fh, lh);
      }
      combine(lo.q, fl, ll, hi.q, fh, lh, f);
      double* dstf = role == 2 ? &sFY[ppar][0][i_slot] : &sFZ[ppar][0][i_slot];
#pragma unroll
      for (int k = 0; k < M; ++k) dstf[k * NIF] = f[k];
    }
    issue(p + 1 + D);
    __syncthreads();
  }

  // ---- next-step dt candidate of the patch (kernels.py:267-281, order 0):
  // per axis a NaN-propagating max over the volumes, then the python max over
  // the axes with NaN axes dropped ----
  if (A.dt_slots) {
    if (nanmask) atomicOr(&sNan, nanmask);
    __syncthreads();
    const unsigned nb = sNan;
    double lmax = 0.0;
#pragma unroll
    for (int a = 0; a < DIM; ++a)
      if (!((nb >> a) & 1u)) lmax = lv[a] > lmax ? lv[a] : lmax;
    unsigned long long key = (unsigned long long)__double_as_longlong(lmax);   // >= 0, NaN-free
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const unsigned long long v = __shfl_xor_sync(0xffffffffu, key, off);
      key = v > key ? v : key;
    }
    if ((tid & 31) == 0 && key) atomicMax(&sLam, key);
    __syncthreads();
    if (tid == 0) {
      const double lam = __longlong_as_double((long long)sLam);
      if (lam > 0.0)
        atomicMin(A.dt_slots + (b % EDG_DT_SLOTS),
                  (unsigned long long)__double_as_longlong(dt_candidate(A.h_cell, 0, lam)));
    }
  }
}

}  // namespace edg
