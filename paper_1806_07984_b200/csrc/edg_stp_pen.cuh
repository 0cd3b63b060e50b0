// Space-time predictor, 2-D "pencil" formulation -- the same Picard iteration
// as stp_picard_kernel (kernels.py:120-159), reorganised so that the operator
// contractions run out of registers with uniform (constant-bank) operators:
//
//   new[r] = c_r q + (-dt/h_0) X_0[r] + (-dt/h_1) X_1[r],
//   X_a[r] = sum_s K^-1[r][s] w_s (D (x)_a F_a(qhat_s))
//
//  * phase A (one thread per spatial node, qhat of its time column in
//    registers): fluxes F_a(qhat_s) for every time node s -> shared memory,
//    in a per-axis layout where each axis-a pencil is strided by N and the
//    pencil index is contiguous;
//  * phase B (one thread per (axis, component, pencil) task): loads the
//    pencil's N x N (time x space) flux block once, contracts space with D
//    and time with K^-1 diag(w) entirely in registers (2 N^3 FMAs per N^2
//    loads; D, K^-1, w are constant-bank operands), and writes X_a in place;
//  * phase A': new iterate, convergence predicate and next fluxes.
// Three barriers per iteration.  The first iteration uses the reduced form
// (qhat_s = q: one flux, X_a[r] = (sum_s K^-1[r][s] w_s) D (x)_a F_a(q)).
// Epilogue, persistent work blocks and the q prefetch are those of
// stp_picard_kernel.  Per-cell exit semantics are identical; the result is a
// different (non-associative) fp64 contraction order, checked against the
// oracle to the same tolerance.
#pragma once
#include "edg_stp.cuh"

namespace edg {

// constant-bank basis table kPen: edg_stp.cuh

template <int KIND, int N>
struct PenCfg {
  static constexpr int DIM = 2;
  static constexpr int M = Pde<KIND, DIM>::M;
  static constexpr int NPC = N * N;
  static constexpr int NF = N;
  static constexpr int TPC = 2 * M * N;                  // phase-B tasks per cell
  static constexpr int PER = (NPC > TPC ? NPC : TPC);   // threads needed per cell
  static constexpr int CPB = PER >= 96 ? 1 : (PER >= 48 ? 4 : (PER >= 24 ? 6 : 8));
  static constexpr int THREADS = ((CPB * PER + 31) / 32) * 32;
  static constexpr int N3 = N * N * N;
  // (axis, component) block stride BS = N (mod 16) doubles: consecutive phase-B
  // tasks (pencils p, then components) hit consecutive bank pairs
  static constexpr int BS = N3 + ((N - N3 % 16) % 16 + 16) % 16;
  static constexpr int CS = 2 * M * BS;                  // flux doubles per cell
  static constexpr int MINB = THREADS <= 128 ? 3 : 2;
  static constexpr size_t BYTES = sizeof(double) * (CPB * CS + 2 * CPB * M * NPC + CPB * N * M * NPC + N) + sizeof(int) * 3 * CPB;
};

template <int KIND, int N, int MINB = PenCfg<KIND, N>::MINB>
__global__ void __launch_bounds__(PenCfg<KIND, N>::THREADS, MINB) stp_pencil_kernel(const StpArgs A) {
  constexpr int DIM = 2;
  using Cf = PenCfg<KIND, N>;
  constexpr int M = Cf::M, NPC = Cf::NPC, NF = Cf::NF, CPB = Cf::CPB, THREADS = Cf::THREADS;
  constexpr int BS = Cf::BS, CS = Cf::CS, TPC = Cf::TPC;
  constexpr int O = pen_off(N);
  // constant-bank operators
  auto cD = [](int i, int j) { return kPen[O + EDG_BASIS_D(N) + i * N + j]; };
  auto cW = [](int s) { return kPen[O + EDG_BASIS_W(N) + s]; };
  auto cTL = [](int j) { return kPen[O + EDG_BASIS_TL(N) + j]; };
  auto cTR = [](int j) { return kPen[O + EDG_BASIS_TR(N) + j]; };
  auto cK = [](int r, int s) { return kPen[O + EDG_BASIS_KINV(N) + r * N + s]; };
  auto cC = [](int r) { return kPen[O + EDG_BASIS_KLIFT(N) + r]; };

  extern __shared__ __align__(16) double smem[];
  double* const sF = smem;                               // [CPB][2][M][N(s)][N][N]
  double* const sQ0 = sF + CPB * CS;                     // [2][CPB][M][NPC]
  double* const sQH = sQ0 + 2 * CPB * M * NPC;          // qhat [CPB][N][M][NPC] (thread-private)
  double* const sWs = sQH + CPB * N * M * NPC;           // [N] sum_s K^-1[r][s] w_s
  int* const sFlag = reinterpret_cast<int*>(sWs + N);    // [3][CPB]: not converged (by iteration parity) x2, active

  const int tid = threadIdx.x;
  const int slot = tid / NPC;
  const int node = tid - slot * NPC;
  const bool lane_ok = slot < CPB;                       // node thread
  const int i0 = node / N, i1 = node - (node / N) * N;
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
  if (tid < N) {
    double ws = 0.0;
#pragma unroll
    for (int s = 0; s < N; ++s) ws = fma(cK(tid, s), cW(s), ws);
    sWs[tid] = ws;
  }

  // node (i0, i1): axis-0 block [k][s][i0][i1], axis-1 block [k][s][i1][i0]
  const int n0 = i0 * N + i1, n1 = i1 * N + i0;
  double* const cellF = sF + slot * CS;
  unsigned its_sum = 0u;

  for (int gi = 0; blk < nblocks; blk += gridDim.x, ++gi) {
    const int item = blk * CPB + slot;
    const bool has_cell = lane_ok && (item < A.nwork);
    const int cell = has_cell ? (A.cell_list ? __ldg(A.cell_list + item) : item) : 0;
    if (blk + (int)gridDim.x < nblocks) prefetch_q(blk + gridDim.x, (gi + 1) & 1);
    cp_async_commit();
    if (tid < CPB) {
      sFlag[tid] = 0;
      sFlag[CPB + tid] = 0;
      sFlag[2 * CPB + tid] = (blk * CPB + tid < A.nwork) ? 1 : 0;
    }
    double sc0 = 0.0, sc1 = 0.0;   // -dt / h_a
    {
      const double* e = A.edges + (A.edges_per_cell ? (size_t)cell * DIM : 0);
      sc0 = -dt / e[0];
      sc1 = -dt / e[1];
    }
    cp_async_wait1();
    const double* const q0s = sQ0 + (gi & 1) * QB + slot * M * NPC + node;
    // qhat of this node's time column lives in shared memory (thread-private)
    double* const qhs = sQH + slot * N * M * NPC + node;
    auto QH = [&](int r, int k) -> double& { return qhs[(r * M + k) * NPC]; };
    bool active = has_cell;
    int its = 0;
    bool conv = false;
    // phase A: fluxes of the time nodes [s_lo, s_hi) -> flux blocks
    auto put_fluxes = [&](int s_count) {
#pragma unroll
      for (int s = 0; s < N; ++s) {
        if (s < s_count) {
          double q[M], F[DIM][M];
#pragma unroll
          for (int k = 0; k < M; ++k) q[k] = (s_count == 1) ? q0s[k * NPC] : QH(s, k);
          FastFlux<KIND, DIM>::template all<M>(q, A.pp, F);
#pragma unroll
          for (int k = 0; k < M; ++k) {
            cellF[k * BS + s * NPC + n0] = F[0][k];
            cellF[(M + k) * BS + s * NPC + n1] = F[1][k];
          }
        }
      }
    };
    if (active) put_fluxes(1);

    for (int it = 1; it <= A.max_iter; ++it) {
      __syncthreads();   // B1: fluxes (and active flags) visible
      // ---- phase B: (cell, axis, component, pencil) tasks ----
      for (int t = tid; t < CPB * TPC; t += THREADS) {
        const int cl = t / TPC;
        if (!sFlag[2 * CPB + cl]) continue;
        const int rem = t - cl * TPC;
        const int p = rem % N;
        const int ak = rem / N;            // a * M + k
        double* const blkp = sF + cl * CS + ak * BS + p;
        double X[N][N];                    // X[r][i]
        if (it == 1) {
          double f[N], y[N];
#pragma unroll
          for (int j = 0; j < N; ++j) f[j] = blkp[j * N];
#pragma unroll
          for (int i = 0; i < N; ++i) {
            double v = 0.0;
#pragma unroll
            for (int j = 0; j < N; ++j) v = fma(cD(i, j), f[j], v);
            y[i] = v;
          }
#pragma unroll
          for (int r = 0; r < N; ++r) {
            const double ws = sWs[r];
#pragma unroll
            for (int i = 0; i < N; ++i) X[r][i] = ws * y[i];
          }
        } else {
#pragma unroll
          for (int r = 0; r < N; ++r)
#pragma unroll
            for (int i = 0; i < N; ++i) X[r][i] = 0.0;
#pragma unroll
          for (int s = 0; s < N; ++s) {
            double f[N], y[N];
#pragma unroll
            for (int j = 0; j < N; ++j) f[j] = blkp[(s * N + j) * N];
#pragma unroll
            for (int i = 0; i < N; ++i) {
              double v = 0.0;
#pragma unroll
              for (int j = 0; j < N; ++j) v = fma(cD(i, j), f[j], v);
              y[i] = v * cW(s);
            }
#pragma unroll
            for (int r = 0; r < N; ++r)
#pragma unroll
              for (int i = 0; i < N; ++i) X[r][i] = fma(cK(r, s), y[i], X[r][i]);
            // keep the next time node's loads below this point (bounded
            // register pressure: X plus one pencil row in flight)
            asm volatile("" ::: "memory");
          }
        }
#pragma unroll
        for (int r = 0; r < N; ++r)
#pragma unroll
          for (int i = 0; i < N; ++i) blkp[(r * N + i) * N] = X[r][i];
      }
      __syncthreads();   // B2: X_a in place
      // ---- phase A': new iterate, convergence predicate ----
      bool below = true;
      if (active) {
#pragma unroll
        for (int k = 0; k < M; ++k) {
          const double q0 = q0s[k * NPC];
#pragma unroll
          for (int r = 0; r < N; ++r) {
            const double x0 = cellF[k * BS + r * NPC + n0];
            const double x1 = cellF[(M + k) * BS + r * NPC + n1];
            const double v = fma(sc1, x1, fma(sc0, x0, cC(r) * q0));
            below = below & (fabs(v - (it == 1 ? q0 : QH(r, k))) < A.tol);
            QH(r, k) = v;
          }
        }
        if (!below) sFlag[(it & 1) * CPB + slot] = 1;
      }
      // B3: the flags are visible, and the CTA continues iff some active cell
      // has a lane not below tol
      const bool any = __syncthreads_or(active && !below);
      if (active) {
        its = it;
        if (sFlag[(it & 1) * CPB + slot] == 0) {
          active = false;
          conv = true;
        }
      }
      // node 0 of each cell republishes the active flag (read by phase B after
      // the next B1) and clears the other parity's flag for the next iteration
      if (lane_ok && node == 0) {
        sFlag[2 * CPB + slot] = active ? 1 : 0;
        sFlag[((it + 1) & 1) * CPB + slot] = 0;
      }
      if (!any) break;
      if (active) put_fluxes(N);
    }

    // ---------------------------------------------------------- epilogue --
    // (as stp_picard_kernel) q_end, q_int, dt-weighted integrated fluxes
    double* St = sF + slot * ((1 + DIM) * M * NPC);
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
        const double tr = cTR(r), w = cW(r);
        double q[M], F[DIM][M];
#pragma unroll
        for (int k = 0; k < M; ++k) q[k] = QH(r, k);
        FastFlux<KIND, DIM>::template all<M>(q, A.pp, F);
#pragma unroll
        for (int k = 0; k < M; ++k) {
          qe[k] = fma(tr, q[k], qe[k]);
          qi[k] = fma(w, q[k], qi[k]);
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
      }
    }
    __syncthreads();
    if (has_cell) {
#pragma unroll
      for (int k = 0; k < M; ++k) St[k * NPC + node] = qi[k];
#pragma unroll
      for (int a = 0; a < DIM; ++a)
#pragma unroll
        for (int k = 0; k < M; ++k) St[((1 + a) * M + k) * NPC + node] = fi[a][k] * dt;
    }
    __syncthreads();
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
        double qa = 0.0, qb = 0.0, fa = 0.0, fb = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j) {
          const double vq = sq[j * st], vf = sf[j * st];
          qa = fma(cTL(j), vq, qa);
          qb = fma(cTR(j), vq, qb);
          fa = fma(cTL(j), vf, fa);
          fb = fma(cTR(j), vf, fb);
        }
        const size_t o0 = tbase + ((size_t)(2 * a) * M + k) * NF + f;
        const size_t o1 = tbase + ((size_t)(2 * a + 1) * M + k) * NF + f;
        A.trace_q[o0] = qa;
        A.trace_q[o1] = qb;
        A.trace_f[o0] = fa;
        A.trace_f[o1] = fb;
      }
    }
    if (has_cell && node == 0) its_sum += (unsigned)its;
    __syncthreads();
  }
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
