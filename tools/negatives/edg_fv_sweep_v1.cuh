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
#define EDG_FV_SWEEP 0
#endif
#ifndef EDG_FV_SWEEP_MINB
#define EDG_FV_SWEEP_MINB 3
#endif

template <int KIND, int DIM, int K>
struct FvSweep {
  static constexpr bool ENABLED = EDG_FV_SWEEP && KIND == EDG_PDE_EULER && DIM == 3 && K == 8;
  static constexpr int COLS = K * K;          // column threads
  static constexpr int HALO = 4 * K;          // halo threads: y+, y-, z+, z- rows of the plane
  static constexpr int THREADS = COLS + HALO;
  static constexpr int NV = 8;                // q[5], 1/rho, p, c
  static constexpr int NIF = (K + 1) * K;     // interfaces of one transverse axis per plane
};

template <int K, int MINB>
__global__ void __launch_bounds__(FvSweep<EDG_PDE_EULER, 3, K>::THREADS, MINB) fv_sweep_kernel(const FvArgs A) {
  const TraceScope trace_scope(A.trace);
  constexpr int KIND = EDG_PDE_EULER, DIM = 3;
  using P = Pde<KIND, DIM>;
  using Cf = FvSweep<KIND, DIM, K>;
  constexpr int M = P::M, NC = K * K * K, NL = K * K;
  constexpr int COLS = Cf::COLS, NV = Cf::NV, NIF = Cf::NIF, SP = Cf::THREADS;
  // halo rows in the plane's state block: y+ first (a warp's upper-y loads of
  // rows 6, 7 and the y+ row then cover 16 distinct bank pairs)
  constexpr int H_YP = COLS, H_YM = COLS + K, H_ZP = COLS + 2 * K, H_ZM = COLS + 3 * K;

  __shared__ double sS[NV][SP];        // states of the current plane (+ parts)
  __shared__ double sFY[M][NIF];       // y interfaces j = 0..K: between rows j-1 and j, [j * K + z]
  __shared__ double sFZ[M][NIF];       // z interfaces: [y * (K + 1) + j]
  __shared__ double sCoef[DIM];
  __shared__ unsigned long long sLam;
  __shared__ unsigned sNan;

  const int tid = threadIdx.x;
  const int b = A.patch_base + (int)blockIdx.x;
  const bool col = tid < COLS;
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
  auto publish = [&](int x, const State& s) {
#pragma unroll
    for (int k = 0; k < M; ++k) sS[k][x] = s.q[k];
    sS[M][x] = s.inv;
    sS[M + 1][x] = s.p;
    sS[M + 2][x] = s.c;
  };
  auto fetch = [&](int x, State& s) {
#pragma unroll
    for (int k = 0; k < M; ++k) s.q[k] = sS[k][x];
    s.inv = sS[M][x];
    s.p = sS[M + 1][x];
    s.c = sS[M + 2][x];
  };
  // F_a(s) and |u_a| + c
  auto flux_of = [&](const State& s, int a, double* f, double& l) {
    const typename P::Parts pr{s.inv, s.p};
    P::flux(s.q, pr, a, A.pp, f);
    l = __dadd_rn(fabs(__dmul_rn(P::mom(s.q, a), s.inv)), s.c);
  };
  // Rusanov flux between lo and hi (kernels.py:162-173), exact order
  auto combine = [&](const State& lo, const double* fl, double ll, const State& hi, const double* fh, double lh,
                     double* f) {
    const double hl = __dmul_rn(0.5, nan_max(ll, lh));
#pragma unroll
    for (int k = 0; k < M; ++k)
      f[k] = __dsub_rn(__dmul_rn(0.5, __dadd_rn(fl[k], fh[k])), __dmul_rn(hl, __dsub_rn(hi.q[k], lo.q[k])));
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

  // ---- per-thread source pointers ----
  // column thread: own planes, and the x-/x+ halo planes; halo thread: its
  // halo state of plane x at hp + x * hxs.  cs = component stride.
  const double* own = A.patch + (size_t)b * M * NC + tid;
  const double *pm = own, *pp_ = own, *hp = own;
  int cs_m = NC, cs_p = NC, hcs = NC, hxs = NL;
  int y = 0, z = 0;                    // column coordinates
  int h_int = 0, h_slot = 0, h_axis = 1, h_hi = 0, h_row = H_YP;
  if (col) {
    y = tid / K;
    z = tid - y * K;
    if (A.halos) {
      pm = A.halos + ((size_t)b * 2 * DIM + 0) * M * NL + tid;
      pp_ = A.halos + ((size_t)b * 2 * DIM + 1) * M * NL + tid;
      cs_m = cs_p = NL;
    } else {
      // neighbour below contributes its last plane, above its first;
      // outflow (-1): own plane on that side (kernels.py:256-264)
      const int nm = neighbour(0, 0), np = neighbour(0, 1);
      pm = A.patch + (size_t)(nm >= 0 ? nm : b) * M * NC + (nm >= 0 ? (K - 1) * NL : 0) + tid;
      pp_ = A.patch + (size_t)(np >= 0 ? np : b) * M * NC + (np >= 0 ? 0 : (K - 1) * NL) + tid;
    }
  } else {
    const int h = tid - COLS, side = h / K, t = h - side * K;   // side: 0 y+, 1 y-, 2 z+, 3 z-
    h_axis = 1 + (side >> 1);
    h_hi = (side & 1) ^ 1;                                      // 1: the halo state is the upper one
    h_row = COLS + side * K + t;
    const int e_in = h_hi ? K - 1 : 0;                          // interior neighbour's coordinate on the axis
    h_int = h_axis == 1 ? e_in * K + t : t * K + e_in;
    h_slot = h_axis == 1 ? (h_hi ? K : 0) * K + t : t * (K + 1) + (h_hi ? K : 0);
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
  // upper neighbours of a column thread in the plane's state block
  const int up_y = y < K - 1 ? tid + K : H_YP + z;
  const int up_z = z < K - 1 ? tid + 1 : H_ZP + y;

  State prev, cur;
  double nxt[M];
  double fxl[M], fxc[M], lxc = 0.0;     // lower x flux of the pending volume; F_0 and wave speed of `prev`
  double dy[M], dz[M];                  // c1 (Fy+ - Fy-), c2 (Fz+ - Fz-) of the pending volume
  double lv[DIM] = {0.0, 0.0, 0.0};
  unsigned nanmask = 0u;
#pragma unroll
  for (int k = 0; k < M; ++k) {
    nxt[k] = col ? __ldg(pm + (size_t)k * cs_m) : __ldg(hp + (size_t)k * hcs);
    prev.q[k] = fxl[k] = fxc[k] = dy[k] = dz[k] = 0.0;
  }
  prev.inv = prev.p = prev.c = 0.0;
  __syncthreads();                      // sCoef, sLam, sNan
  const double c0 = sCoef[0], c1 = sCoef[1], c2 = sCoef[2];

#pragma unroll 1
  for (int x = -1; x <= K; ++x) {
    const bool inner = x >= 0 && x < K;
    if (col) {
#pragma unroll
      for (int k = 0; k < M; ++k) cur.q[k] = nxt[k];
      if (x < K) {
        const double* src = x + 1 < K ? own + (x + 1) * NL : pp_;
        const int cs = x + 1 < K ? NC : cs_p;
#pragma unroll
        for (int k = 0; k < M; ++k) nxt[k] = __ldg(src + (size_t)k * cs);
      }
      eval_parts(cur);
      double fc[M], lc;
      flux_of(cur, 0, fc, lc);
      if (x >= 0) {
        double fxh[M];
        combine(prev, fxc, lxc, cur, fc, lc, fxh);          // interface x - 1/2
        if (x >= 1) {
          // volume x - 1 of this column is complete
          double o[M];
          bool finite = true;
          double* dst = A.out + (size_t)b * M * NC + (x - 1) * NL + tid;
#pragma unroll
          for (int k = 0; k < M; ++k) {
            o[k] = __dsub_rn(prev.q[k], __dmul_rn(c0, __dsub_rn(fxh[k], fxl[k])));
            o[k] = __dsub_rn(o[k], dy[k]);
            o[k] = __dsub_rn(o[k], dz[k]);
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
#pragma unroll
        for (int k = 0; k < M; ++k) fxl[k] = fxh[k];
      }
#pragma unroll
      for (int k = 0; k < M; ++k) fxc[k] = fc[k];
      lxc = lc;
      if (inner) publish(tid, cur);
    } else if (inner) {
#pragma unroll
      for (int k = 0; k < M; ++k) cur.q[k] = nxt[k];
      if (x + 1 < K) {
#pragma unroll
        for (int k = 0; k < M; ++k) nxt[k] = __ldg(hp + (size_t)(x + 1) * hxs + (size_t)k * hcs);
      }
      eval_parts(cur);
      publish(h_row, cur);
    }
    if (!inner) {
      if (col) prev = cur;
      continue;
    }
    __syncthreads();                    // the plane's states are published
    if (col) {
      State nb;
      double fl[M], ll, fh[M], lh, f[M];
      flux_of(cur, 1, fl, ll);
      fetch(up_y, nb);
      flux_of(nb, 1, fh, lh);
      combine(cur, fl, ll, nb, fh, lh, f);
      if (y < K - 1) {
#pragma unroll
        for (int k = 0; k < M; ++k) sFY[k][tid + K] = f[k];
      }
      flux_of(cur, 2, fl, ll);
      fetch(up_z, nb);
      flux_of(nb, 2, fh, lh);
      combine(cur, fl, ll, nb, fh, lh, f);
      if (z < K - 1) {
#pragma unroll
        for (int k = 0; k < M; ++k) sFZ[k][y * (K + 1) + z + 1] = f[k];
      }
    } else {
      State in;
      double fa[M], la, fb[M], lb, f[M];
      fetch(h_int, in);
      flux_of(in, h_axis, fa, la);
      flux_of(cur, h_axis, fb, lb);
      if (h_hi) combine(in, fa, la, cur, fb, lb, f);
      else combine(cur, fb, lb, in, fa, la, f);
      double* dstf = h_axis == 1 ? &sFY[0][h_slot] : &sFZ[0][h_slot];
#pragma unroll
      for (int k = 0; k < M; ++k) dstf[k * NIF] = f[k];
    }
    __syncthreads();                    // the plane's y / z fluxes are published
    if (col) {
#pragma unroll
      for (int k = 0; k < M; ++k) {
        dy[k] = __dmul_rn(c1, __dsub_rn(sFY[k][tid + K], sFY[k][tid]));
        dz[k] = __dmul_rn(c2, __dsub_rn(sFZ[k][y * (K + 1) + z + 1], sFZ[k][y * (K + 1) + z]));
      }
      prev = cur;
    }
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
