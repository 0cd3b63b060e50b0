// 2-D space-time predictor (Picard), plane formulation -- replaces
// kernels.py:120-159 for 2-D Euler cells of n = 4 nodes per axis (EDG_STP2_MAXN).
//
// The per-node kernel of edg_stp.cuh contracts both spatial derivatives in the
// thread of the node: 2 n flux loads per component and time node, 2 stores,
// and four barriers per iteration.  Here (as in the 3-D kernel's plane tasks,
// edg_stp3.cuh) a full iteration of a cell runs in three phases over all n
// time nodes, two barriers apart.  It ships for n = 4 (config 5 / 1's order),
// where the n m = 16 plane tasks of a cell are exactly its 16 node threads;
// at n = 6 it measured 35 % slower than the per-node kernel (EDG_STP2_MAXN).
//
//   A  node threads: F_0(qhat_s), F_1(qhat_s) of their node for every s into
//      the rows [a][s][k] of the cell's flux block (natural node order);
//   B  plane tasks (time node s, component k), one per thread, n m <= n^2 of
//      them per cell: F_0's n x n plane in registers, F_1 streamed row by row,
//          H[i0][i1] = sum_l D[i0][l] F_0[l][i1] + sum_l D[i1][l] F_1[i0][l]
//      (D a constant-bank operand) written over F_1's row -- every flux value
//      is read once;
//   C  node threads: dv = H at their node, time contraction
//      acc[r] += K^-1[r][s] (-dt w_s) dv.
//
// Shared-memory accesses per node and (time node, component): 2 + 3 + 1 = 6
// instead of 2 n + 2.  The reduced first iteration (one time node) keeps the
// node-local derivative (its n m plane tasks would occupy m threads per
// cell).  Cells of a CTA converge independently (per-cell flags, as in
// edg_stp.cuh); the epilogue is that kernel's.  1/h: cells whose two edges
// are equal (every cell of a uniform or 3:1-refined mesh) fold it into the
// time coefficients; a work block with an anisotropic cell scales the two
// derivative sums inside the plane task.
#pragma once
#include <type_traits>

#include "edg_stp.cuh"

#ifndef EDG_STP2_PLANE
#define EDG_STP2_PLANE 1
#endif
// resident CTAs per SM asked of ptxas
#ifndef EDG_STP2_MINB
#define EDG_STP2_MINB(n) ((n) <= 4 ? 6 : ((n) == 5 ? 3 : 2))
#endif
// node threads per CTA aimed at (cells per CTA = the best fill of whole warps below it)
// (cfg5, n = 4: 4 cells in 64 threads at 6 CTAs per SM, 160 registers: 36 us for
// the two launches; 6 cells in 96 threads 38 us; 8 in 128 threads 44-49 us;
// 2 in 32 threads 37-40 us; the per-node kernel 40 us)
#ifndef EDG_STP2_TARGET
#define EDG_STP2_TARGET 64
#endif
// largest n that takes this kernel (n = 6 measured 35 % slower than the
// per-node kernel on cfg2: 255 registers, 2 CTAs per SM, 24 of 36 lanes in
// the plane phase)
#ifndef EDG_STP2_MAXN
#define EDG_STP2_MAXN 4
#endif

namespace edg {

template <int KIND, int N>
struct Stp2Cfg {
  static constexpr int M = Pde<KIND, 2>::M;
  static constexpr int NPC = N * N;
  static constexpr bool ENABLED = EDG_STP2_PLANE != 0 && KIND == EDG_PDE_EULER && N >= 4 && N <= EDG_STP2_MAXN && N * M <= NPC;
  static constexpr int CPB = stp_best_cpb(NPC, EDG_STP2_TARGET);
  static constexpr int THREADS = ((CPB * NPC + 31) / 32) * 32;
  static constexpr int ROW = NPC | 1;                       // odd row stride: 16 consecutive rows on 16 bank pairs
  static constexpr int CELL0 = 2 * N * M * ROW;             // rows [a][s][k] of one cell
  // cell stride = n^2 (mod 16): a warp's node accesses run on across a cell boundary
  static constexpr int CELL = CELL0 + (((NPC - CELL0) % 16) + 16) % 16;
  static constexpr int OPS = N * N + 2 * N + (N & 1);       // D, K^-1 lift, sum_s B[r][s] (even)
  static constexpr size_t BYTES = sizeof(double) * (OPS + CPB * CELL + 2 * CPB * M * NPC) + sizeof(int) * 2 * CPB;
  static constexpr int MINB = EDG_STP2_MINB(N);
  static_assert(CELL >= 3 * M * NPC, "epilogue staging must fit a cell's flux block");
};

template <int KIND, int N>
__global__ void __launch_bounds__(Stp2Cfg<KIND, N>::THREADS, Stp2Cfg<KIND, N>::MINB)
stp_picard2_kernel(const StpArgs A) {
  const TraceScope trace_scope(A.trace);
  using Cf = Stp2Cfg<KIND, N>;
  constexpr int DIM = 2;
  constexpr int M = Cf::M, NPC = Cf::NPC, NF = N, CPB = Cf::CPB, THREADS = Cf::THREADS, ROW = Cf::ROW, CELL = Cf::CELL;
  constexpr int O = pen_off(N);   // this order's block in the constant-bank operator table

  extern __shared__ __align__(16) double smem[];
  double* sD = smem;                          // D[N][N] (first iteration: rows indexed by the node)
  double* sC = sD + N * N;                    // K^-1 lift
  double* sBs = sC + N;                       // sum_s B[r][s]
  double* sF = smem + Cf::OPS;                // [CPB][a][s][k][ROW]
  double* sQ0 = sF + CPB * CELL;              // initial state [2][CPB][M][NPC] (thread-private)
  int* sFlag = reinterpret_cast<int*>(sQ0 + 2 * CPB * M * NPC);   // [2][CPB] "not converged" flags

  const int tid = threadIdx.x;
  const int slot = tid / NPC;
  const int node = tid - slot * NPC;
  const bool lane_ok = slot < CPB;
  const int i0 = node / N, i1 = node - i0 * N;
  double* const cF = sF + (lane_ok ? slot : 0) * CELL;       // this cell's rows
  auto row = [&](int a, int g, int k) -> int { return ((a * N + g) * M + k) * ROW; };
  // plane task of this thread: (time node, component) = (node / M, node % M)
  const bool task_ok = lane_ok && node < N * M;
  const int tg = task_ok ? node / M : 0, tk = task_ok ? node - tg * M : 0;

  const double dt = *A.dt;
  const int nblocks = (A.nwork + CPB - 1) / CPB;
  constexpr int QB = CPB * M * NPC;
  auto prefetch_q = [&](int b, int buf) {
    const int itm = b * CPB + slot;
    if (lane_ok && itm < A.nwork) {
      const int c = A.cell_list ? __ldg(A.cell_list + itm) : itm;
      const double* src = A.q + (size_t)c * M * NPC + node;
      double* dst = sQ0 + buf * QB + slot * M * NPC + node;
#pragma unroll
      for (int k = 0; k < M; ++k) cp_async8(dst + k * NPC, src + k * NPC);
    }
  };
  int blk = blockIdx.x;
  if (blk < nblocks) prefetch_q(blk, 0);
  cp_async_commit();
  for (int i = tid; i < N * N; i += THREADS) sD[i] = A.basis[EDG_BASIS_D(N) + i];
  for (int i = tid; i < N; i += THREADS) {
    sC[i] = A.basis[EDG_BASIS_KLIFT(N) + i];
    double bs = 0.0;
    for (int s = 0; s < N; ++s) bs += A.basis[EDG_BASIS_KINV(N) + i * N + s] * (-dt * A.basis[EDG_BASIS_W(N) + s]);
    sBs[i] = bs;
  }
  if (tid < 2 * CPB) sFlag[tid] = 0;
  unsigned its_sum = 0u;

  for (int gi = 0; blk < nblocks; blk += gridDim.x, ++gi) {
    const int item = blk * CPB + slot;
    const bool has_cell = lane_ok && item < A.nwork;
    const int cell = has_cell ? (A.cell_list ? __ldg(A.cell_list + item) : item) : 0;
    if (blk + (int)gridDim.x < nblocks) prefetch_q(blk + gridDim.x, (gi + 1) & 1);
    cp_async_commit();
    if (tid < 2 * CPB) sFlag[tid] = 0;   // (the previous block's flag reads precede its epilogue barrier)
    // 1/h of this thread's cell; the block folds it into the time coefficients
    // when every cell of the block is isotropic
    const double* e = A.edges + (A.edges_per_cell ? (size_t)cell * DIM : 0);
    const double ih0 = 1.0 / e[0], ih1 = 1.0 / e[1];
    cp_async_wait1();   // this block's initial state (own node) has landed
    // (barrier: operators and flags settled, the previous block's epilogue reads done)
    const bool iso = __syncthreads_and(!has_cell || e[0] == e[1]) != 0;
    const double ihc = iso ? ih0 : 1.0;

    const double* const q0s = sQ0 + (gi & 1) * QB + (lane_ok ? slot : 0) * M * NPC + node;
    double qh[N][M], acc[N][M];
#pragma unroll
    for (int k = 0; k < M; ++k) {
      const double v = has_cell ? q0s[k * NPC] : 1.0;
#pragma unroll
      for (int r = 0; r < N; ++r) qh[r][k] = v;
    }
    bool active = has_cell;
    int its = 0;
    bool conv = false, inacc = false;
    const int max_iter = A.max_iter;

    // A: flux of time node g at this node -> rows [a][g][k]
    auto put_flux = [&](int g, const double* q) {
      double F[DIM][M];
      FastFlux<KIND, DIM>::template all<M>(q, A.pp, F);
#pragma unroll
      for (int a = 0; a < DIM; ++a)
#pragma unroll
        for (int k = 0; k < M; ++k) cF[row(a, g, k) + node] = F[a][k];
    };
    // B: this thread's plane task, H over F_1's row
    auto plane = [&](auto scaled) {
      constexpr bool SC = decltype(scaled)::value;
      const double* P0 = cF + row(0, tg, tk);
      double* P1 = cF + row(1, tg, tk);
      double f0[N][N];
#pragma unroll
      for (int l = 0; l < N; ++l)
#pragma unroll
        for (int j = 0; j < N; ++j) f0[l][j] = P0[l * N + j];
#pragma unroll
      for (int i = 0; i < N; ++i) {
        double f1[N], o[N];
#pragma unroll
        for (int l = 0; l < N; ++l) f1[l] = P1[i * N + l];
#pragma unroll
        for (int j = 0; j < N; ++j) {
          double h0 = 0.0, h1 = 0.0;
#pragma unroll
          for (int l = 0; l < N; ++l) {
            h0 = fma(kPen[O + EDG_BASIS_D(N) + i * N + l], f0[l][j], h0);
            h1 = fma(kPen[O + EDG_BASIS_D(N) + j * N + l], f1[l], h1);
          }
          o[j] = SC ? fma(h0, ih0, h1 * ih1) : h0 + h1;
        }
#pragma unroll
        for (int j = 0; j < N; ++j) P1[i * N + j] = o[j];
      }
    };
    // per-cell exit (kernels.py:143-147): "every |new - qhat| < tol" per thread,
    // a per-cell flag, one barrier; the CTA goes on while some cell is active
    auto finish = [&](int it, bool below, bool into_acc) -> bool {
      int* flag = sFlag + (it & 1) * CPB;
      if (active && !below) flag[slot] = 1;
      const bool any = __syncthreads_or(active && !below);
      if (active) {
        its = it;
        inacc = into_acc;
        if (flag[slot] == 0) {
          active = false;
          conv = true;
        }
      }
      if (tid < CPB) sFlag[((it + 1) & 1) * CPB + tid] = 0;
      return any;
    };

    bool any = false;
    if (max_iter >= 1) {
      // reduced first iteration: qhat_s = q for every s (kernels.py:134), so
      //   acc[r] = c_r q + (sum_s B[r][s]) div F(q), node-local derivative
      if (active) {
        double q[M];
#pragma unroll
        for (int k = 0; k < M; ++k) q[k] = qh[0][k];
        put_flux(0, q);
      }
      __syncthreads();
      bool below = true;
      if (active) {
#pragma unroll
        for (int k = 0; k < M; ++k) {
          const double* F0 = cF + row(0, 0, k) + i1;
          const double* F1 = cF + row(1, 0, k) + i0 * N;
          double h0 = 0.0, h1 = 0.0;
#pragma unroll
          for (int j = 0; j < N; ++j) {
            h0 = fma(sD[i0 * N + j], F0[j * N], h0);
            h1 = fma(sD[i1 * N + j], F1[j], h1);
          }
          const double dv = iso ? (h0 + h1) * ihc : fma(h0, ih0, h1 * ih1);
#pragma unroll
          for (int r = 0; r < N; ++r) {
            acc[r][k] = fma(sBs[r], dv, sC[r] * qh[r][k]);
            below = below & (fabs(acc[r][k] - qh[r][k]) < A.tol);
          }
        }
      }
      any = finish(1, below, true);
    }
    // full iteration: qn = c q + sum_s B[r][s] div F(qc_s); returns "some cell goes on"
    auto body = [&](const double (&qc)[N][M], double (&qn)[N][M], int it, bool into_acc) -> bool {
      if (active) {
#pragma unroll
        for (int g = 0; g < N; ++g) {
          double q[M];
#pragma unroll
          for (int k = 0; k < M; ++k) q[k] = qc[g][k];
          put_flux(g, q);
        }
      }
      __syncthreads();
      if (active && task_ok) {
        if (iso)
          plane(std::false_type{});
        else
          plane(std::true_type{});
      }
      __syncthreads();
      bool below = true;
      if (active) {
#pragma unroll
        for (int k = 0; k < M; ++k) {
          const double q0 = q0s[k * NPC];
#pragma unroll
          for (int r = 0; r < N; ++r) qn[r][k] = kPen[O + EDG_BASIS_KLIFT(N) + r] * q0;
        }
#pragma unroll
        for (int g = 0; g < N; ++g) {
          double dv[M];
#pragma unroll
          for (int k = 0; k < M; ++k) dv[k] = cF[row(1, g, k) + node];
          const double sc = -(dt * kPen[O + EDG_BASIS_W(N) + g]) * ihc;   // (-dt) w_s (/ h when isotropic)
#pragma unroll
          for (int r = 0; r < N; ++r) {
            const double b = kPen[O + EDG_BASIS_KINV(N) + r * N + g] * sc;
#pragma unroll
            for (int k = 0; k < M; ++k) qn[r][k] = fma(b, dv[k], qn[r][k]);
          }
        }
#pragma unroll
        for (int r = 0; r < N; ++r)
#pragma unroll
          for (int k = 0; k < M; ++k) below = below & (fabs(qn[r][k] - qc[r][k]) < A.tol);
      }
      return finish(it, below, into_acc);   // the barrier also guards the rows for the next iteration
    };
    for (int it = 2; any && it <= max_iter;) {
      any = body(acc, qh, it, false);
      if (!any || ++it > max_iter) break;
      any = body(qh, acc, it, true);
      ++it;
    }
    if (inacc) {
#pragma unroll
      for (int r = 0; r < N; ++r)
#pragma unroll
        for (int k = 0; k < M; ++k) qh[r][k] = acc[r][k];
    }

    // ---------------------------------------------------------- epilogue --
    // q_end = sum_r l_r(1) qhat_r; q_int = dt sum_r w_r qhat_r;
    // fint_a = dt sum_r w_r F_a(qhat_r)          (kernels.py:148-155),
    // staged as [(1 + d) m][n^2] in the cell's block for the face projections
    double* St = cF;
    double qe[M], qi[M], fi[DIM][M];
#pragma unroll
    for (int k = 0; k < M; ++k) qe[k] = qi[k] = 0.0;
#pragma unroll
    for (int a = 0; a < DIM; ++a)
#pragma unroll
      for (int k = 0; k < M; ++k) fi[a][k] = 0.0;
    if (has_cell) {
#pragma unroll
      for (int r = 0; r < N; ++r) {
        const double tr = kPen[O + EDG_BASIS_TR(N) + r], w = kPen[O + EDG_BASIS_W(N) + r];
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
        its_sum += (unsigned)its;
      }
      // (the last finish() barrier ordered every read of the rows before these stores)
#pragma unroll
      for (int k = 0; k < M; ++k) St[k * NPC + node] = qi[k];
#pragma unroll
      for (int a = 0; a < DIM; ++a)
#pragma unroll
        for (int k = 0; k < M; ++k) St[((1 + a) * M + k) * NPC + node] = fi[a][k] * dt;
    }
    __syncthreads();
    // face projections, one task per (axis a, face point f): both sides of
    // trace_q and trace_f for every component (kernels.py:73-79, 148-157)
    for (int task = node; has_cell && task < DIM * NF; task += NPC) {
      constexpr int PER_FAM = 2 * DIM * M * NF;
      const size_t tbase = (size_t)cell * PER_FAM;
      const int a = task / NF, f = task - a * NF;
      const int st = a == DIM - 1 ? 1 : N;
      const int base = a == DIM - 1 ? f * N : f;
#pragma unroll
      for (int k = 0; k < M; ++k) {
        const double* sq = St + k * NPC + base;
        const double* sf = St + ((1 + a) * M + k) * NPC + base;
        double q0 = 0.0, q1 = 0.0, f0 = 0.0, f1 = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j) {
          const double vq = sq[j * st], vf = sf[j * st];
          q0 = fma(kPen[O + EDG_BASIS_TL(N) + j], vq, q0);
          q1 = fma(kPen[O + EDG_BASIS_TR(N) + j], vq, q1);
          f0 = fma(kPen[O + EDG_BASIS_TL(N) + j], vf, f0);
          f1 = fma(kPen[O + EDG_BASIS_TR(N) + j], vf, f1);
        }
        const size_t o0 = tbase + ((size_t)(2 * a) * M + k) * NF + f;
        const size_t o1 = tbase + ((size_t)(2 * a + 1) * M + k) * NF + f;
        A.trace_q[o0] = q0;
        A.trace_q[o1] = q1;
        A.trace_f[o0] = f0;
        A.trace_f[o1] = f1;
      }
    }
    // (the next block's first barrier orders these staging reads before its flux writes)
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
