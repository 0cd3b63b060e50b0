// Space-time predictor, node-pair / time-split kernel for 2-D even node
// counts (configs 1, 2, 5) -- same algorithm as edg_stp.cuh
// (kernels.py:120-159), different thread -> work map.
//
// Why: the one-thread-per-node kernel is bound by shared-memory wavefronts
// (every derivative FMA needs its own LDS: 36 loads per 48 FMAs per node and
// time node; ncu: 0.71 wavefronts/clk/SM with the FP64 pipe at 39 %).  Here a
// lane pair owns two adjacent nodes n0 = (i, 2jp), n1 = (i, 2jp + 1) of a row:
//   * lane h = 0 holds time nodes 0..H-1, lane h = 1 time nodes H..N-1
//     (H = N/2) of both nodes: qhat and the next iterate in registers;
//   * every 16-byte load of a flux buffer feeds both nodes: on axis 0 the pair
//     (F[l][2jp], F[l][2jp+1]) is one LDS.128 used by the two columns, on
//     axis 1 the row pencil F[i][2l..2l+1] is shared by both nodes, so one
//     LDS.128 feeds four FMAs (36 LDS.128 per 96 FMAs instead of 36 per 48);
//   * flux values are stored as 16-byte pairs;
//   * per pipeline stage t each lane contracts the derivative of its own time
//     node s_h = h*H + t, swaps it with the partner (shfl.xor 1) and applies
//     both time columns of B = K^-1 diag(-dt w) to its own rows:
//         acc[r] += B[r][s_own] div_own + B[r][s_par] div_par
//     so an iteration has H barriers;
//   * the flux of the next iteration's first time node is evaluated
//     speculatively before the convergence barrier, which doubles as the last
//     stage's barrier;
//   * the iteration loop is unrolled by two so qhat and the next iterate swap
//     roles without register moves.
// The first Picard iteration uses qhat_s = q for every s (kernels.py:134):
// one flux, one derivative (split by component between the two lanes) and
// acc[r] = c_r q + (sum_s B[r][s]) div F(q), as in edg_stp.cuh.
#pragma once
#include "edg_stp.cuh"

namespace edg {

template <int N>
struct StpPairCfg {
  static constexpr int NPC = N * N;
  static constexpr int H = N / 2;
#ifndef EDG_PAIR_TARGET
#define EDG_PAIR_TARGET 160
#endif
  static constexpr int CPB = stp_best_cpb(NPC, EDG_PAIR_TARGET);
  static constexpr int THREADS = ((CPB * NPC + 31) / 32) * 32;
#ifndef EDG_PAIR_MINB
#define EDG_PAIR_MINB 2
#endif
  static constexpr int MINB = EDG_PAIR_MINB;
};

template <int KIND, int N>
struct StpPairSmem {
  using C = StpPairCfg<N>;
  static constexpr int M = Pde<KIND, 2>::M;
  static constexpr int NPC = N * N;
  static constexpr int OPS = 2 * N * N + 6 * N;   // KP pairs, D, c, Bs, w, tl, tr (+pad)
  static constexpr int SS = 2 * M * NPC;          // one cell's flux of one time node [a][k][node]
  static constexpr int FB0 = C::CPB * SS;
  // (stage, half) buffer stride = 8 (mod 16) doubles: the two halves of a
  // warp read the same relative words 16 banks apart
  static constexpr int FB = FB0 + ((8 - FB0 % 16) + 16) % 16;
  static constexpr int QB = C::CPB * M * NPC;
  static_assert(C::CPB * 3 * M * NPC <= 4 * FB, "epilogue staging must fit in the flux buffers");
  static constexpr size_t BYTES = sizeof(double) * (OPS + 4 * FB + 2 * QB) + sizeof(int) * 3 * C::CPB;
};

template <int KIND, int N, int MINB = StpPairCfg<N>::MINB>
__global__ void __launch_bounds__(StpPairCfg<N>::THREADS, MINB)
stp_pair_kernel(const StpArgs A) {
  static_assert(N % 2 == 0, "node-pair predictor needs an even node count");
  using P = Pde<KIND, 2>;
  using Cf = StpPairCfg<N>;
  using Sm = StpPairSmem<KIND, N>;
  constexpr int M = P::M;
  constexpr int NPC = Cf::NPC, NF = N, CPB = Cf::CPB, THREADS = Cf::THREADS, H = Cf::H;
  constexpr int PAIRS = NPC / 2;
  constexpr int MH = (M + 1) / 2;   // components per lane in the first iteration

  extern __shared__ __align__(16) double smem[];
  double2* sKP = reinterpret_cast<double2*>(smem);   // [h][t][rho] = (B[r][s_own], B[r][s_par])
  double* sD = smem + N * N;                         // D[N][N]
  double* sC = sD + N * N;                           // K^-1 lift
  double* sBs = sC + N;                              // sum_s B[r][s]
  double* sW = sBs + N;
  double* sTL = sW + N;
  double* sTR = sTL + N;
  double* sF = smem + Sm::OPS;                       // [stage 2][half 2] x FB
  double* sQ0 = sF + 4 * Sm::FB;                     // initial state [2][CPB][M][NPC]
  int* sFlag = reinterpret_cast<int*>(sQ0 + 2 * Sm::QB);   // [3][CPB] "not converged" flags

  const int tid = threadIdx.x;
  const int h = tid & 1;
  const int slot = (tid >> 1) / PAIRS;
  const int pr = (tid >> 1) - slot * PAIRS;
  const int i0 = pr / H;               // row (axis-0 index) of the pair
  const int jp = pr - i0 * H;          // pair index along axis 1
  const int n0 = i0 * N + 2 * jp;      // nodes n0, n0 + 1
  const int lt = tid - slot * NPC;     // lane index within the cell (face tasks)
  const bool lane_ok = slot < CPB;
  const double dt = *A.dt;

  const int nblocks = (A.nwork + CPB - 1) / CPB;
  constexpr int QB = Sm::QB;
  // the pair's initial state (both nodes, 16-byte pieces), components split
  // between the two lanes; visible to the partner after wait + __syncwarp
  auto prefetch_q = [&](int b, int buf) {
    const int itm = b * CPB + slot;
    if (lane_ok && itm < A.nwork) {
      const int c = A.cell_list ? __ldg(A.cell_list + itm) : itm;
      const double* src = A.q + (size_t)c * M * NPC + n0;
      double* dst = sQ0 + buf * QB + slot * M * NPC + n0;
#pragma unroll
      for (int k = 0; k < M; ++k)
        if ((k & 1) == h) cp_async16(dst + k * NPC, src + k * NPC);
    }
  };
  int blk = blockIdx.x;
  if (blk < nblocks) prefetch_q(blk, 0);
  cp_async_commit();

  for (int i = tid; i < N * N; i += THREADS) sD[i] = A.basis[EDG_BASIS_D(N) + i];
  // B[r][s] = K^-1[r][s] * ((-dt) * w[s]) exactly as edg_stp.cuh folds it
  auto Bv = [&](int r, int s) { return A.basis[EDG_BASIS_KINV(N) + r * N + s] * (-dt * A.basis[EDG_BASIS_W(N) + s]); };
  for (int i = tid; i < 2 * H * H; i += THREADS) {
    const int hh = i / (H * H), t = (i / H) % H, rho = i % H;
    const int r = hh * H + rho;
    sKP[i] = make_double2(Bv(r, hh * H + t), Bv(r, (1 - hh) * H + t));
  }
  for (int i = tid; i < N; i += THREADS) {
    sW[i] = A.basis[EDG_BASIS_W(N) + i];
    sTL[i] = A.basis[EDG_BASIS_TL(N) + i];
    sTR[i] = A.basis[EDG_BASIS_TR(N) + i];
    sC[i] = A.basis[EDG_BASIS_KLIFT(N) + i];
    double bs = 0.0;
    for (int s = 0; s < N; ++s) bs += Bv(i, s);
    sBs[i] = bs;
  }
  __syncthreads();

  unsigned its_sum = 0u;
  for (int gi = 0; blk < nblocks; blk += gridDim.x, ++gi) {
    const int item = blk * CPB + slot;
    const bool has_cell = lane_ok && (item < A.nwork);
    const int cell = has_cell ? (A.cell_list ? __ldg(A.cell_list + item) : item) : 0;
    if (blk + (int)gridDim.x < nblocks) prefetch_q(blk + gridDim.x, (gi + 1) & 1);
    cp_async_commit();
    if (tid < 3 * CPB) sFlag[tid] = 0;
    // derivative rows scaled by 1/h_a: axis 0 row i0 (shared by the pair),
    // axis 1 rows 2jp and 2jp + 1
    double Dr0[N], Dr1[2][N];
    {
      const double* e = A.edges + (A.edges_per_cell ? (size_t)cell * 2 : 0);
      const double ih0 = 1.0 / e[0], ih1 = 1.0 / e[1];
#pragma unroll
      for (int l = 0; l < N; ++l) {
        Dr0[l] = sD[i0 * N + l] * ih0;
        Dr1[0][l] = sD[(2 * jp) * N + l] * ih1;
        Dr1[1][l] = sD[(2 * jp + 1) * N + l] * ih1;
      }
    }
    cp_async_wait1();
    __syncwarp();
    const double* const q0s = sQ0 + (gi & 1) * QB + slot * M * NPC + n0;
    auto load_q0 = [&](double (&q)[2][M]) {
#pragma unroll
      for (int k = 0; k < M; ++k) {
        const double2 v = has_cell ? *reinterpret_cast<const double2*>(q0s + k * NPC) : make_double2(1.0, 1.0);
        q[0][k] = v.x;
        q[1][k] = v.y;
      }
    };
    auto fbuf = [&](int p, int hh) { return sF + (p * 2 + hh) * Sm::FB + slot * Sm::SS; };
    // flux of one time node at both nodes -> [a][k][node] as 16-byte pairs
    auto put_flux = [&](double* Fb, const double (&q)[2][M]) {
      double F0[2][M], F1[2][M];
      FastFlux<KIND, 2>::template all<M>(q[0], A.pp, F0);
      FastFlux<KIND, 2>::template all<M>(q[1], A.pp, F1);
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int k = 0; k < M; ++k)
          *reinterpret_cast<double2*>(Fb + (a * M + k) * NPC + n0) = make_double2(F0[a][k], F1[a][k]);
    };
    // axis-0 part of component k at both nodes: column pair (2jp, 2jp+1)
    auto d_axis0 = [&](const double* Fb, int k, double& a0, double& a1) {
      const double* f = Fb + k * NPC + 2 * jp;
#pragma unroll
      for (int l = 0; l < N; ++l) {
        const double2 v = *reinterpret_cast<const double2*>(f + l * N);
        a0 = fma(Dr0[l], v.x, a0);
        a1 = fma(Dr0[l], v.y, a1);
      }
    };
    // axis-1 part of component k at both nodes: row pencil i0, shared
    auto d_axis1 = [&](const double* Fb, int k, double& a0, double& a1) {
      const double* f = Fb + (M + k) * NPC + i0 * N;
#pragma unroll
      for (int l = 0; l < N; l += 2) {
        const double2 v = *reinterpret_cast<const double2*>(f + l);
        a0 = fma(Dr1[0][l], v.x, a0);
        a0 = fma(Dr1[0][l + 1], v.y, a0);
        a1 = fma(Dr1[1][l], v.x, a1);
        a1 = fma(Dr1[1][l + 1], v.y, a1);
      }
    };
    // div F at both nodes, all components: per-axis chains summed (the
    // one-thread-per-node kernel's order)
    auto deriv = [&](const double* Fb, double (&dv)[2][M]) {
#pragma unroll
      for (int k = 0; k < M; ++k) {
        double x0 = 0.0, x1 = 0.0, y0 = 0.0, y1 = 0.0;
        d_axis0(Fb, k, x0, x1);
        d_axis1(Fb, k, y0, y1);
        dv[0][k] = x0 + y0;
        dv[1][k] = x1 + y1;
      }
    };

    double qA[H][2][M], qB[H][2][M];
    bool active = has_cell;
    int its = 0;
    bool conv = false;
    bool finB = true;   // the latest iterate is in qB (else qA)
    int g = 0;          // pipeline stage counter: flux buffer parity
    const int max_iter = A.max_iter;

    auto finish_iteration = [&](int it, bool below, bool intoB) -> bool {
      int* flag = sFlag + (it % 3) * CPB;
      if (active && !below) flag[slot] = 1;
      const bool any = __syncthreads_or(active && !below);
      ++g;
      if (active) {
        its = it;
        finB = intoB;
        if (flag[slot] == 0) {
          active = false;
          conv = true;
        }
      }
      // parity it+2 was last read before this barrier and is next written
      // after the next one
      if (tid < CPB) sFlag[((it + 2) % 3) * CPB + tid] = 0;
      return any;
    };

    bool any = false;
    if (max_iter < 1) {
      double q[2][M];
      load_q0(q);
#pragma unroll
      for (int r = 0; r < H; ++r)
#pragma unroll
        for (int n = 0; n < 2; ++n)
#pragma unroll
          for (int k = 0; k < M; ++k) qB[r][n][k] = q[n][k];
    } else {
      // ---------------------------------------------- first iteration --
      double q[2][M];
      load_q0(q);
      double* Fb = fbuf(0, 0);
      if (active) {
        double F0[2][M], F1[2][M];
        FastFlux<KIND, 2>::template all<M>(q[0], A.pp, F0);
        FastFlux<KIND, 2>::template all<M>(q[1], A.pp, F1);
        // lane h stores the flux components k = h, h + 2, ...
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int k = 0; k < M; ++k)
            if ((k & 1) == h) *reinterpret_cast<double2*>(Fb + (a * M + k) * NPC + n0) = make_double2(F0[a][k], F1[a][k]);
      }
      __syncthreads();
      // lane h contracts components k = 2kk + h, then the pair swaps
      double mine[2][MH];
#pragma unroll
      for (int kk = 0; kk < MH; ++kk) {
        const int k = 2 * kk + h;
        double x0 = 0.0, x1 = 0.0, y0 = 0.0, y1 = 0.0;
        if (active && k < M) {
          d_axis0(Fb, k, x0, x1);
          d_axis1(Fb, k, y0, y1);
        }
        mine[0][kk] = x0 + y0;
        mine[1][kk] = x1 + y1;
      }
      double dv[2][M];
#pragma unroll
      for (int kk = 0; kk < MH; ++kk)
#pragma unroll
        for (int n = 0; n < 2; ++n) {
          const double other = __shfl_xor_sync(0xffffffffu, mine[n][kk], 1);
          if (2 * kk < M) dv[n][2 * kk] = h ? other : mine[n][kk];
          if (2 * kk + 1 < M) dv[n][2 * kk + 1] = h ? mine[n][kk] : other;
        }
      bool below = true;
      if (active) {
#pragma unroll
        for (int r = 0; r < H; ++r) {
          const double c = sC[h * H + r], b = sBs[h * H + r];
#pragma unroll
          for (int n = 0; n < 2; ++n)
#pragma unroll
            for (int k = 0; k < M; ++k) {
              const double v = fma(b, dv[n][k], c * q[n][k]);
              below = below & (fabs(v - q[n][k]) < A.tol);
              qB[r][n][k] = v;
            }
        }
        put_flux(fbuf(1, h), qB[0]);   // speculative: next iteration's first stage
      }
      any = finish_iteration(1, below, true);
    }

    // ------------------------------------------- iterations 2, 3, ... --
    // entry: fbuf(g & 1, h) holds the flux of qc[0] of this lane's half
    auto body = [&](const double (&qc)[H][2][M], double (&qn)[H][2][M], int it, bool intoB) -> bool {
      if (active) {
        double q[2][M];
        load_q0(q);
#pragma unroll
        for (int r = 0; r < H; ++r) {
          const double c = sC[h * H + r];
#pragma unroll
          for (int n = 0; n < 2; ++n)
#pragma unroll
            for (int k = 0; k < M; ++k) qn[r][n][k] = c * q[n][k];
        }
      }
#pragma unroll
      for (int t = 0; t < H; ++t) {
        if (active && t + 1 < H) put_flux(fbuf((g + 1) & 1, h), qc[t + 1]);
        double dvo[2][M];
        if (active) deriv(fbuf(g & 1, h), dvo);
        double dvp[2][M];
#pragma unroll
        for (int n = 0; n < 2; ++n)
#pragma unroll
          for (int k = 0; k < M; ++k) dvp[n][k] = __shfl_xor_sync(0xffffffffu, dvo[n][k], 1);
        if (active) {
#pragma unroll
          for (int r = 0; r < H; ++r) {
            const double2 b = sKP[(h * H + t) * H + r];
#pragma unroll
            for (int n = 0; n < 2; ++n)
#pragma unroll
              for (int k = 0; k < M; ++k) qn[r][n][k] = fma(b.y, dvp[n][k], fma(b.x, dvo[n][k], qn[r][n][k]));
          }
        }
        if (t + 1 < H) {
          __syncthreads();
          ++g;
        }
      }
      bool below = true;
      if (active) {
#pragma unroll
        for (int r = 0; r < H; ++r)
#pragma unroll
          for (int n = 0; n < 2; ++n)
#pragma unroll
            for (int k = 0; k < M; ++k) below = below & (fabs(qn[r][n][k] - qc[r][n][k]) < A.tol);
        put_flux(fbuf((g + 1) & 1, h), qn[0]);   // speculative
      }
      return finish_iteration(it, below, intoB);
    };

    for (int it = 2; any && it <= max_iter;) {
      any = body(qB, qA, it, false);
      if (!any || ++it > max_iter) break;
      any = body(qA, qB, it, true);
      ++it;
    }

    // ------------------------------------------------------- epilogue --
    // partial sums over this lane's time nodes, completed with the partner's
    double qe[2][M], qi[2][M], fi[2][2][M];
#pragma unroll
    for (int n = 0; n < 2; ++n)
#pragma unroll
      for (int k = 0; k < M; ++k) {
        qe[n][k] = qi[n][k] = 0.0;
        fi[n][0][k] = fi[n][1][k] = 0.0;
      }
    if (has_cell) {
#pragma unroll
      for (int r = 0; r < H; ++r) {
        const double tr = sTR[h * H + r], w = sW[h * H + r];
#pragma unroll
        for (int n = 0; n < 2; ++n) {
          double q[M];
#pragma unroll
          for (int k = 0; k < M; ++k) q[k] = finB ? qB[r][n][k] : qA[r][n][k];
          double F[2][M];
          FastFlux<KIND, 2>::template all<M>(q, A.pp, F);
#pragma unroll
          for (int k = 0; k < M; ++k) {
            qe[n][k] = fma(tr, q[k], qe[n][k]);
            qi[n][k] = fma(w, q[k], qi[n][k]);
            fi[n][0][k] = fma(w, F[0][k], fi[n][0][k]);
            fi[n][1][k] = fma(w, F[1][k], fi[n][1][k]);
          }
        }
      }
    }
    // own + partner (commutative: both lanes get the same bits); lane h keeps node n0 + h
    double qe_h[M], qi_h[M], fi_h[2][M];
#pragma unroll
    for (int k = 0; k < M; ++k) {
      double s[2], u[2], f0[2], f1[2];
#pragma unroll
      for (int n = 0; n < 2; ++n) {
        s[n] = qe[n][k] + __shfl_xor_sync(0xffffffffu, qe[n][k], 1);
        u[n] = qi[n][k] + __shfl_xor_sync(0xffffffffu, qi[n][k], 1);
        f0[n] = fi[n][0][k] + __shfl_xor_sync(0xffffffffu, fi[n][0][k], 1);
        f1[n] = fi[n][1][k] + __shfl_xor_sync(0xffffffffu, fi[n][1][k], 1);
      }
      qe_h[k] = h ? s[1] : s[0];
      qi_h[k] = (h ? u[1] : u[0]) * dt;
      fi_h[0][k] = h ? f0[1] : f0[0];
      fi_h[1][k] = h ? f1[1] : f1[0];
    }
    const int node = n0 + h;
    if (has_cell) {
      double* qend = A.q_end + (size_t)cell * M * NPC + node;
      double* qint = A.q_int ? A.q_int + (size_t)cell * M * NPC + node : nullptr;
#pragma unroll
      for (int k = 0; k < M; ++k) {
        qend[k * NPC] = qe_h[k];
        if (qint) qint[k * NPC] = qi_h[k];
      }
      if (lt == 0) {
        A.iterations[cell] = its;
        A.converged[cell] = conv ? 1 : 0;
      }
    }
    // the flux buffers may still be read by other cells' last iteration until here
    __syncthreads();
    double* St = sF + slot * (3 * M * NPC);
    if (has_cell) {
#pragma unroll
      for (int k = 0; k < M; ++k) St[k * NPC + node] = qi_h[k];
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int k = 0; k < M; ++k) St[((1 + a) * M + k) * NPC + node] = fi_h[a][k] * dt;
    }
    __syncthreads();
    // face projections, one task per (axis a, pencil f) (as in edg_stp.cuh)
    constexpr int TASKS = 2 * NF;
    for (int task = lt; has_cell && task < TASKS; task += NPC) {
      constexpr int PER_FAM = 4 * M * NF;
      const size_t tbase = (size_t)cell * PER_FAM;
      const int a = task / NF, f = task - a * NF;
      const int st = a == 1 ? 1 : N;
      const int base = a == 1 ? f * N : f;
#pragma unroll
      for (int k = 0; k < M; ++k) {
        const double* sq = St + k * NPC + base;
        const double* sf = St + ((1 + a) * M + k) * NPC + base;
        double q0 = 0.0, q1 = 0.0, f0 = 0.0, f1 = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j) {
          const double vq = sq[j * st], vf = sf[j * st];
          q0 = fma(sTL[j], vq, q0);
          q1 = fma(sTR[j], vq, q1);
          f0 = fma(sTL[j], vf, f0);
          f1 = fma(sTR[j], vf, f1);
        }
        const size_t o0 = tbase + ((size_t)(2 * a) * M + k) * NF + f;
        const size_t o1 = tbase + ((size_t)(2 * a + 1) * M + k) * NF + f;
        A.trace_q[o0] = q0;
        A.trace_q[o1] = q1;
        A.trace_f[o0] = f0;
        A.trace_f[o1] = f1;
      }
    }
    if (has_cell && lt == 0) its_sum += (unsigned)its;
    __syncthreads();
  }  // work blocks
  if (A.iter_total) {
    __shared__ unsigned int sIts;
    if (tid == 0) sIts = 0u;
    __syncthreads();
    if (its_sum) atomicAdd(&sIts, its_sum);
    __syncthreads();
    if (tid == 0 && sIts) atomicAdd(A.iter_total, (unsigned long long)sIts);
  }
}

}  // namespace edg
