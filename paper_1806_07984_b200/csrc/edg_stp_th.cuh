// Space-time predictor, time-split variant for even node counts (2-D p = 3,
// 5, 7; configs 1, 2, 5) -- same algorithm as edg_stp.cuh (kernels.py:120-159).
//
// Two threads per spatial node: thread (node, h) owns the time nodes
// r = h*N/2 .. h*N/2 + N/2 - 1 of the node's column (qhat and the next
// iterate in registers, half the registers of the one-thread-per-node
// kernel, hence twice the resident warps).  Per pipeline step s both threads
// store the flux of their time node s_h = h*N/2 + s, contract its spatial
// derivative from shared memory, swap the derivative with the partner lane
// (shfl.xor 16) and apply both time columns of K^-1 to their own rows:
//     acc[r] += B[r][s_0] div_{s_0} + B[r][s_1] div_{s_1}
// so one iteration needs N/2 barriers instead of N.  Warp w covers the 16
// CTA-nodes 16w..16w+15 (lanes 0-15: h = 0, lanes 16-31: h = 1).
#pragma once
#include "edg_stp.cuh"

namespace edg {

template <int DIM, int N>
struct StpThCfg {
  static constexpr int NPC = ipow(N, DIM);
  static constexpr int NF = ipow(N, DIM - 1);
  static constexpr int H = N / 2;
  // cells per CTA: ~128-160 nodes, a multiple of 16 nodes when possible
  static constexpr int CPB = NPC >= 64 ? 1 : (NPC == 36 ? 2 : 64 / NPC);
  static constexpr int NODES = CPB * NPC;
  static constexpr int WARPS = (NODES + 15) / 16;
  static constexpr int THREADS = WARPS * 32;
  static constexpr int MINB = 3;
};

template <int KIND, int DIM, int N>
struct StpThSmem {
  using C = StpThCfg<DIM, N>;
  static constexpr int M = Pde<KIND, DIM>::M;
  static constexpr int OPS = 2 * N * N + 6 * N;
  static constexpr int FH = C::CPB * DIM * M * C::NPC;          // flux of one time node, all cells
  static constexpr size_t BYTES = sizeof(double) * (OPS + 4 * FH) + sizeof(unsigned long long) * 2 * C::CPB;
};

template <int KIND, int DIM, int N>
__global__ void __launch_bounds__(StpThCfg<DIM, N>::THREADS, StpThCfg<DIM, N>::MINB)
stp_picard_th_kernel(const StpArgs A) {
  static_assert(N % 2 == 0, "time-split predictor needs an even node count");
  using P = Pde<KIND, DIM>;
  using Cf = StpThCfg<DIM, N>;
  using Sm = StpThSmem<KIND, DIM, N>;
  constexpr int M = P::M;
  constexpr int NPC = Cf::NPC, NF = Cf::NF, CPB = Cf::CPB, H = Cf::H, THREADS = Cf::THREADS;

  extern __shared__ __align__(16) double smem[];
  double* sD = smem;                 // D[N][N]
  double* sB = sD + N * N;           // B[r][s] = K^-1[r][s] * (-dt w_s)
  double* sW = sB + N * N;
  double* sTL = sW + N;
  double* sTR = sTL + N;
  double* sC = sTR + N;              // K^-1 lift
  double* sBs = sC + N;              // sum_s B[r][s]
  double* sF = smem + Sm::OPS;       // [2 (pipeline)][2 (h)][CPB][DIM][M][NPC]
  unsigned long long* sRed = reinterpret_cast<unsigned long long*>(sF + 4 * Sm::FH);   // [2][CPB]

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int h = lane >> 4;
  const int gnode = (tid >> 5) * 16 + (lane & 15);
  const int slot = gnode / NPC;
  const int node = gnode - slot * NPC;
  const int item = blockIdx.x * CPB + slot;
  const bool has_cell = (gnode < Cf::NODES) && (item < A.nwork);
  const int cell = has_cell ? (A.cell_list ? __ldg(A.cell_list + item) : item) : 0;
  const double dt = *A.dt;

  for (int i = tid; i < N * N; i += THREADS) {
    sD[i] = A.basis[EDG_BASIS_D(N) + i];
    sB[i] = A.basis[EDG_BASIS_KINV(N) + i] * (-dt * A.basis[EDG_BASIS_W(N) + i % N]);
  }
  for (int i = tid; i < N; i += THREADS) {
    sW[i] = A.basis[EDG_BASIS_W(N) + i];
    sTL[i] = A.basis[EDG_BASIS_TL(N) + i];
    sTR[i] = A.basis[EDG_BASIS_TR(N) + i];
    sC[i] = A.basis[EDG_BASIS_KLIFT(N) + i];
    double bs = 0.0;
    for (int s = 0; s < N; ++s) bs += A.basis[EDG_BASIS_KINV(N) + i * N + s] * (-dt * A.basis[EDG_BASIS_W(N) + s]);
    sBs[i] = bs;
  }
  for (int i = tid; i < 2 * CPB; i += THREADS) sRed[i] = 0ull;
  __syncthreads();

  int ix[DIM];
  {
    int t = node;
#pragma unroll
    for (int a = DIM - 1; a >= 0; --a) {
      ix[a] = t % N;
      t /= N;
    }
  }
  int pb[DIM];
#pragma unroll
  for (int a = 0; a < DIM; ++a) pb[a] = node - ix[a] * ipow(N, DIM - 1 - a);
  double Dr[DIM][N];
  {
    const double* e = A.edges + (A.edges_per_cell ? (size_t)cell * DIM : 0);
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
      const double ih = 1.0 / e[a];
#pragma unroll
      for (int j = 0; j < N; ++j) Dr[a][j] = sD[ix[a] * N + j] * ih;
    }
  }

  const double* qsrc = A.q + (size_t)cell * M * NPC + node;
  double qh[H][M], acc[H][M];
#pragma unroll
  for (int k = 0; k < M; ++k) {
    const double v = has_cell ? __ldg(qsrc + k * NPC) : 1.0;
#pragma unroll
    for (int r = 0; r < H; ++r) qh[r][k] = v;
  }

  bool active = has_cell;
  int its = 0;
  bool conv = false;
  const int max_iter = A.max_iter;
  // flux buffer of pipeline stage p for half hh
  auto fbuf = [&](int p, int hh) { return sF + (p * 2 + hh) * Sm::FH + slot * (DIM * M * NPC); };

  auto put_flux = [&](double* Fb, const double* q) {
    double F[DIM][M];
    FastFlux<KIND, DIM>::template all<M>(q, A.pp, F);
#pragma unroll
    for (int a = 0; a < DIM; ++a)
#pragma unroll
      for (int k = 0; k < M; ++k) Fb[(a * M + k) * NPC + node] = F[a][k];
  };
  auto deriv = [&](const double* Fb, double (&dv)[M]) {
    double part[DIM][M];
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
      const int st = ipow(N, DIM - 1 - a);
#pragma unroll
      for (int k = 0; k < M; ++k) {
        const double* Fa = Fb + (a * M + k) * NPC + pb[a];
        double acc_ak = 0.0;
        if (a == DIM - 1) {
#pragma unroll
          for (int j = 0; j < N; j += 2) {
            const double2 v = *reinterpret_cast<const double2*>(Fa + j);
            acc_ak = fma(Dr[a][j], v.x, acc_ak);
            acc_ak = fma(Dr[a][j + 1], v.y, acc_ak);
          }
        } else {
#pragma unroll
          for (int j = 0; j < N; ++j) acc_ak = fma(Dr[a][j], Fa[j * st], acc_ak);
        }
        part[a][k] = acc_ak;
      }
    }
#pragma unroll
    for (int k = 0; k < M; ++k) {
      double v = part[0][k];
#pragma unroll
      for (int a = 1; a < DIM; ++a) v += part[a][k];
      dv[k] = v;
    }
  };

  for (int it = 1; it <= max_iter; ++it) {
    if (it == 1) {
      // qhat_s = q for all s: one flux (stored by h = 0), one derivative
      if (active && h == 0) put_flux(fbuf(0, 0), qh[0]);
      __syncthreads();
      if (active) {
        double dv[M];
        deriv(fbuf(0, 0), dv);
#pragma unroll
        for (int k = 0; k < M; ++k)
#pragma unroll
          for (int r = 0; r < H; ++r) acc[r][k] = fma(sBs[h * H + r], dv[k], sC[h * H + r] * qh[r][k]);
      }
    } else {
      if (active) {
#pragma unroll
        for (int k = 0; k < M; ++k) {
          const double q0 = __ldg(qsrc + k * NPC);
#pragma unroll
          for (int r = 0; r < H; ++r) acc[r][k] = sC[h * H + r] * q0;
        }
        put_flux(fbuf(0, h), qh[0]);
      }
      __syncthreads();
#pragma unroll
      for (int s = 0; s < H; ++s) {
        double dv[M], dp[M];
        if (active) {
          if (s + 1 < H) put_flux(fbuf((s + 1) & 1, h), qh[s + 1]);
          deriv(fbuf(s & 1, h), dv);
        } else {
#pragma unroll
          for (int k = 0; k < M; ++k) dv[k] = 0.0;
        }
        // partner lane (other half of the same node) holds time node s of the other half
#pragma unroll
        for (int k = 0; k < M; ++k) dp[k] = __shfl_xor_sync(0xffffffffu, dv[k], 16);
        if (active) {
          const int s_own = h * H + s, s_oth = (1 - h) * H + s;
#pragma unroll
          for (int r = 0; r < H; ++r) {
            const double b_own = sB[(h * H + r) * N + s_own];
            const double b_oth = sB[(h * H + r) * N + s_oth];
#pragma unroll
            for (int k = 0; k < M; ++k) acc[r][k] = fma(b_oth, dp[k], fma(b_own, dv[k], acc[r][k]));
          }
        }
        __syncthreads();
      }
    }
    unsigned long long* red = sRed + (it & 1) * CPB;
    unsigned long long mk = 0ull;
    if (active) {
#pragma unroll
      for (int r = 0; r < H; ++r)
#pragma unroll
        for (int k = 0; k < M; ++k) {
          const unsigned long long key = maxkey(fabs(acc[r][k] - qh[r][k]));
          mk = key > mk ? key : mk;
          qh[r][k] = acc[r][k];
        }
    }
    {
      const unsigned long long o = __shfl_xor_sync(0xffffffffu, mk, 16);
      mk = o > mk ? o : mk;
    }
    seg_max_atomic(red, (h == 0 && gnode < Cf::NODES) ? slot : -1, mk);
    __syncthreads();
    if (active) {
      its = it;
      const double delta = from_maxkey(red[slot]);
      if (delta < A.tol) {
        active = false;
        conv = true;
      }
    }
    if (tid < CPB) sRed[((it + 1) & 1) * CPB + tid] = 0ull;
    if (!__syncthreads_or(active)) break;
  }

  // ---------------------------------------------------------- epilogue --
  double qe[M], qi[M], fi[DIM][M];
#pragma unroll
  for (int k = 0; k < M; ++k) qe[k] = qi[k] = 0.0;
#pragma unroll
  for (int a = 0; a < DIM; ++a)
#pragma unroll
    for (int k = 0; k < M; ++k) fi[a][k] = 0.0;
  if (has_cell) {
#pragma unroll
    for (int r = 0; r < H; ++r) {
      const double tr = sTR[h * H + r], w = sW[h * H + r];
      double F[DIM][M];
      FastFlux<KIND, DIM>::template all<M>(qh[r], A.pp, F);
#pragma unroll
      for (int k = 0; k < M; ++k) {
        qe[k] = fma(tr, qh[r][k], qe[k]);
        qi[k] = fma(w, qh[r][k], qi[k]);
      }
#pragma unroll
      for (int a = 0; a < DIM; ++a)
#pragma unroll
        for (int k = 0; k < M; ++k) fi[a][k] = fma(w, F[a][k], fi[a][k]);
    }
  }
  // combine the two halves of the time sums
#pragma unroll
  for (int k = 0; k < M; ++k) {
    qe[k] += __shfl_xor_sync(0xffffffffu, qe[k], 16);
    qi[k] += __shfl_xor_sync(0xffffffffu, qi[k], 16);
  }
#pragma unroll
  for (int a = 0; a < DIM; ++a)
#pragma unroll
    for (int k = 0; k < M; ++k) fi[a][k] += __shfl_xor_sync(0xffffffffu, fi[a][k], 16);
  double* St = sF + slot * ((1 + DIM) * M * NPC);
  if (has_cell && h == 0) {
    double* qend = A.q_end + (size_t)cell * M * NPC + node;
    double* qint = A.q_int ? A.q_int + (size_t)cell * M * NPC + node : nullptr;
#pragma unroll
    for (int k = 0; k < M; ++k) {
      qi[k] *= dt;
      qend[k * NPC] = qe[k];
      if (qint) qint[k * NPC] = qi[k];
    }
    if (node == 0) {
      A.iterations[cell] = its;
      A.converged[cell] = conv ? 1 : 0;
    }
  }
  __syncthreads();
  if (has_cell && h == 0) {
#pragma unroll
    for (int k = 0; k < M; ++k) St[k * NPC + node] = qi[k];
#pragma unroll
    for (int a = 0; a < DIM; ++a)
#pragma unroll
      for (int k = 0; k < M; ++k) St[((1 + a) * M + k) * NPC + node] = fi[a][k] * dt;
  }
  __syncthreads();
  if (has_cell) {
    constexpr int PER_FAM = 2 * DIM * M * NF;
    const size_t tbase = (size_t)cell * PER_FAM;
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
      constexpr int dummy = 0;
      (void)dummy;
      const int st = ipow(N, DIM - 1 - a);
      constexpr int ITEMS = 2 * 2 * M * NF;
      for (int o = node + h * NPC; o < ITEMS; o += 2 * NPC) {
        const int f = o % NF;
        const int k = (o / NF) % M;
        const int s = (o / (NF * M)) & 1;
        const int fam = o / (2 * NF * M);
        const int hi = f / st, lo = f - hi * st;
        const double* src = St + ((fam == 0 ? 0 : (1 + a) * M) + k) * NPC + hi * st * N + lo;
        const double* tv = s ? sTR : sTL;
        double v = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j) v = fma(tv[j], src[j * st], v);
        (fam == 0 ? A.trace_q : A.trace_f)[tbase + ((2 * a + s) * M + k) * NF + f] = v;
      }
    }
  }
  if (A.iter_total) {
    __shared__ unsigned int sIts;
    if (tid == 0) sIts = 0u;
    __syncthreads();
    if (has_cell && h == 0 && node == 0) atomicAdd(&sIts, (unsigned)its);
    __syncthreads();
    if (tid == 0 && sIts) atomicAdd(A.iter_total, (unsigned long long)sIts);
  }
}

}  // namespace edg
