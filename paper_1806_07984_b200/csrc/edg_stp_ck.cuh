// Cauchy-Kowalevski space-time predictor for linear PDEs -- replaces
// kernels.py:82-106 (stp_linear).  SURVEY.md section 8(f) row f1.
//
// One thread per spatial node, CPB cells per CTA (same mapping as the Picard
// kernel).  The recurrence term_k = -div F(term_{k-1}) (exact on the tensor
// polynomial space for a linear flux, terminating after d*p terms) runs with
// the term of the node in registers and the flux of the previous term staged
// in shared memory for the derivative contractions:
//     q_end = q + sum_k dt^k / k! term_k
//     q_int = dt q + sum_k dt^(k+1) / (k+1)! term_k
// The epilogue projects q_int onto the faces (trace_q) and, as the reference
// does, evaluates the flux of those traces pointwise (trace_f = F(trace_q)).
#pragma once
#include "edg_stp.cuh"

namespace edg {

template <int KIND, int DIM, int N>
__global__ void __launch_bounds__(StpCfg<DIM, N>::THREADS) stp_linear_kernel(const StpArgs A) {
  using P = Pde<KIND, DIM>;
  using Cf = StpCfg<DIM, N>;
  constexpr int M = P::M;
  constexpr int NPC = Cf::NPC, NF = Cf::NF, CPB = Cf::CPB, THREADS = Cf::THREADS;

  extern __shared__ __align__(16) double smem[];
  double* sD = smem;                                  // D[N][N]
  double* sTL = sD + N * N;
  double* sTR = sTL + N;
  double* sF = sTR + N + (N & 1);                     // [CPB][DIM][M][NPC]; reused for staging

  const int tid = threadIdx.x;
  const int slot = tid / NPC;
  const int node = tid - slot * NPC;
  const int item = blockIdx.x * CPB + slot;
  const bool has_cell = (slot < CPB) && (item < A.nwork);
  const int cell = has_cell ? (A.cell_list ? __ldg(A.cell_list + item) : item) : 0;
  const double dt = *A.dt;
  for (int i = tid; i < N * N; i += THREADS) sD[i] = A.basis[EDG_BASIS_D(N) + i];
  for (int i = tid; i < N; i += THREADS) {
    sTL[i] = A.basis[EDG_BASIS_TL(N) + i];
    sTR[i] = A.basis[EDG_BASIS_TR(N) + i];
  }
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
  double term[M], qe[M], qi[M];
  const size_t cb = (size_t)cell * M * NPC;
#pragma unroll
  for (int k = 0; k < M; ++k) {
    term[k] = has_cell ? __ldg(A.q + cb + (size_t)k * NPC + node) : 0.0;
    qe[k] = term[k];
    qi[k] = dt * term[k];
  }
  double* Fb = sF + slot * (DIM * M * NPC);
  double fact = 1.0, dtk = 1.0;
  for (int kk = 1; kk <= DIM * (N - 1); ++kk) {
    if (has_cell) {
      const auto pr = P::parts(term, A.pp);
#pragma unroll
      for (int a = 0; a < DIM; ++a) {
        double f[M];
        P::flux(term, pr, a, A.pp, f);
#pragma unroll
        for (int k = 0; k < M; ++k) Fb[(a * M + k) * NPC + node] = f[k];
      }
    }
    __syncthreads();
    if (has_cell) {
      fact *= kk;
      dtk *= dt;
      const double c1 = dtk / fact, c2 = dtk * dt / (fact * (kk + 1));
#pragma unroll
      for (int k = 0; k < M; ++k) {
        double dv = 0.0;
#pragma unroll
        for (int a = 0; a < DIM; ++a) {
          const int st = ipow(N, DIM - 1 - a);
          const double* Fa = Fb + (a * M + k) * NPC + (node - ix[a] * st);
#pragma unroll
          for (int j = 0; j < N; ++j) dv = fma(Dr[a][j], Fa[j * st], dv);
        }
        term[k] = -dv;
        qe[k] = fma(c1, term[k], qe[k]);
        qi[k] = fma(c2, term[k], qi[k]);
      }
    }
    __syncthreads();
  }
  if (has_cell) {
#pragma unroll
    for (int k = 0; k < M; ++k) {
      A.q_end[cb + (size_t)k * NPC + node] = qe[k];
      if (A.q_int) A.q_int[cb + (size_t)k * NPC + node] = qi[k];
      Fb[k * NPC + node] = qi[k];
    }
    if (node == 0) {
      A.iterations[cell] = 0;
      A.converged[cell] = 1;
    }
  }
  __syncthreads();
  if (has_cell) {
    // trace_q(a,s)[k][f] = sum_j l_j(s) q_int[k][node(f,a,j)]; trace_f = F_a(trace_q) pointwise
    const size_t tbase = (size_t)cell * 2 * DIM * M * NF;
    for (int o = node; o < 2 * DIM * NF; o += NPC) {
      const int fs = o / NF, f = o - fs * NF;
      const int a = fs >> 1, s = fs & 1;
      const int st = ipow(N, DIM - 1 - a);
      const int hi = f / st, lo = f - hi * st;
      const double* tv = s ? sTR : sTL;
      double tq[M];
#pragma unroll
      for (int k = 0; k < M; ++k) {
        const double* src = Fb + k * NPC + hi * st * N + lo;
        double v = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j) v = fma(tv[j], src[j * st], v);
        tq[k] = v;
        A.trace_q[tbase + ((size_t)fs * M + k) * NF + f] = v;
      }
      const auto pr = P::parts(tq, A.pp);
      double tf[M];
      P::flux(tq, pr, a, A.pp, tf);
#pragma unroll
      for (int k = 0; k < M; ++k) A.trace_f[tbase + ((size_t)fs * M + k) * NF + f] = tf[k];
    }
  }
}

}  // namespace edg
