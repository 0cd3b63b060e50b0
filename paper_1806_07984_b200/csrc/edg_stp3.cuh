// 3-D space-time predictor (Picard), pencil formulation -- replaces
// kernels.py:120-159 for 3-D cells of n >= 5 nodes per axis (one cell per CTA).
//
// The per-node kernel of edg_stp.cuh contracts every spatial derivative in
// the thread of the node it belongs to: 3 axes x n loads of the flux per
// component and time node, which made it shared-memory bound (ncu on cfg3:
// the derivative loads were 38 % of the instructions and ~48 % of the stall
// samples, 2.3 wavefronts per LDS.64).  Here one iteration of a cell runs in
// three phases per group of G time nodes:
//
//   A  node threads: flux F_a(qhat_s) of their node for s in the group,
//      stored into the rows [a][s][k] of the flux buffer, each axis in its own
//      pencil-contiguous layout (node (i0,i1,i2) at n * pencil_a + i_a);
//   B  pencil tasks (axis a, time node s, component k, pencil p): load the n
//      flux values of the pencil, contract them with D (a constant-bank
//      operand, so no register or shared load per FMA) and write
//      (D F)/h_a back in place -- each flux value is read by exactly one task;
//   C  node threads: dv = (H_0 + H_1) + H_2 at their node and the time
//      contraction acc[r] += K^-1[r][s] (-dt w_s) dv.
//
// Shared-memory traffic per full iteration and cell drops from
// 3 n^(d+1) m loads + d n^(d+1) m stores to 2 (d n^(d+1) m) loads + stores
// (cfg3: 56k -> 37.5k accesses), and every pencil access is a stride-n lane
// pattern that the row stride n^3 (= 13 mod 16 for n = 5) keeps at the ideal
// two wavefronts per warp.  The Picard exit test, the exact reduced first
// iteration, the persistent CTAs with cp.async prefetch and the epilogue are
// those of edg_stp.cuh.
#pragma once
#include <type_traits>

#include "edg_stp.cuh"

#ifndef EDG_STP3_ISO
#define EDG_STP3_ISO 1
#endif

namespace edg {

// time nodes per phase group (all five at n = 5: 85 KB of shared memory and
// 2 CTAs per SM; three for larger n so the rows stay under ~80 KB)
#ifndef EDG_STP3_G
#define EDG_STP3_G(n) ((n) <= 5 ? (n) : 3)
#endif
// pencil phase with one (component, pencil) per thread (n = 5; larger n spill)
#ifndef EDG_STP3_KMAP
#define EDG_STP3_KMAP(n) ((n) <= 5)
#endif
// resident CTAs per SM asked of ptxas (n = 5: 248 registers, no spills)
#ifndef EDG_STP3_MINB
#define EDG_STP3_MINB(n) ((n) <= 5 ? 2 : 1)
#endif

// axis-0 rows in the natural node order (node (i0,i1,i2) at n^2 i0 + n i1 +
// i2: unit-stride node-phase accesses, pencil p = n i1 + i2 at p + n^2 j)
// with the row stride padded (n = 5: 137) so the pencil phase's component
// change inside a warp stays conflict-free; 0 = pencil-contiguous like axes 1, 2
#ifndef EDG_STP3_A0NAT
#define EDG_STP3_A0NAT 1
#endif
// axis-1 rows likewise with i1 slowest (node at n^2 i1 + n i2 + i0, pencil
// p = n i2 + i0 at p + n^2 j), row stride as axis 0's
#ifndef EDG_STP3_A1NAT
#define EDG_STP3_A1NAT 1
#endif

// n = 5, axis 1 (EDG_STP3_A1TAB): rows in the natural node order too (unit-
// stride node phase) with row stride 133 (= 5 mod 16); the pencil-phase task
// of thread t is kA1Task[t] = 25 k + 5 i0 + i2 (component k, pencil (i0, i2),
// elements at 25 i0 + i2 + 5 j): the 125 tasks are grouped so that every
// half-warp's 16 tasks fall on 16 distinct 8-byte bank pairs (bank =
// (5 k + 25 i0 + i2) mod 16 has 8 or 7 tasks per bank; half-warp g takes
// the g-th task of each bank) -- conflict-free in both phases
#ifndef EDG_STP3_A1TAB
#define EDG_STP3_A1TAB 1
#endif
static __constant__ signed char kA1Task[128] = {
    0,   1,   2,   3,   4,   13,  14,  23,  24,  5,   6,   7,   8,   9,   18,  19,  32,  33,  10,  11,  12,  21,
    22,  27,  28,  29,  38,  15,  16,  17,  30,  31,  40,  41,  34,  43,  20,  25,  26,  35,  36,  37,  46,  39,
    48,  49,  54,  63,  64,  73,  42,  55,  44,  57,  58,  59,  68,  45,  50,  47,  52,  53,  62,  71,  72,  77,
    74,  79,  56,  65,  66,  67,  80,  69,  82,  51,  60,  61,  70,  75,  76,  85,  78,  87,  88,  89,  98,  99,
    104, 81,  90,  83,  84,  93,  94,  107, 108, 109, 86,  95,  96,  97,  102, 103, 112, 113, 114, 91,  92,  105,
    106, 115, 116, 117, 118, 119, 100, 101, 110, 111, 120, 121, 122, 123, 124, -1,  -1,  -1};


// EDG_STP3_PLANE (n = 5, full iterations): the derivatives along axes 1 and 2
// are contracted together by PLANE tasks -- task (g, k, i0) loads the 5 x 5
// plane i0 of the rows F_1[g][k] and F_2[g][k] (both in natural node order,
// 25 contiguous values each), forms
//     H12[i1][i2] = sum_l D[i1][l] F_1[l][i2] + sum_l D[i2][l] F_2[i1][l]
// with F_1's plane held in registers and F_2 streamed row by row, and writes
// H12 over F_2's plane (row i1 is stored right after it was consumed).  There
// are G M n = 125 plane tasks, one per thread; axis 0 keeps its pencil tasks.
// Shared-memory accesses per node and (time node, component): flux stores 3,
// plane 2 + 1, axis-0 pencils 1 + 1, derivative loads 2 = 10 instead of the
// pencil formulation's 12 -- the kernel is bound by shared-memory wavefronts
// (DESIGN.md section 4).  Both rows then use the stride n^3 = 125 (= 13 mod
// 16, a task's base lands on bank pair (13 (5 g + k) + 9 i0) mod 16, at most 8
// tasks per pair); kPlaneTask assigns the tasks to lanes so that the 16 tasks
// of every half-warp sit on 16 distinct bank pairs, and kA1Task125 does the
// same for the axis-1 pencil tasks of the reduced first iteration (task
// 25 k + 5 i0 + i2 at bank pair (13 k + 9 i0 + i2) mod 16).
#ifndef EDG_STP3_PLANE
#define EDG_STP3_PLANE 1
#endif
static __constant__ signed char kPlaneTask[128] = {
    124, 38, 84, 41, 50, 43, 119, 21, 74, 16, 24, 113, 51, 45, 14, 79, 4, 121, 82, 7, 101, 22, 96, 33, 10,
    35, 11, 104, 76, 93, 110, 47, 36, 39, 105, 86, 85, 81, 59, 66, 19, 64, 88, 42, 44, 78, 61, 31, 20, 9, 6,
    5, 65, 103, 107, 18, 122, 80, 56, 28, 67, 46, 109, 95, 73, 52, 123, 87, 118, 117, 90, 99, 1, 112, 2, 40,
    92, 94, 111, 13, 25, 68, 71, 53, 58, 70, 27, 34, 0, 115, 49, 12, 120, 30, 29, 63, 23, 37, 116, 54, 91,
    106, 114, 89, 3, 48, 60, 8, 97, 77, 62, 15, 69, 75, 98, 55, 26, 100, 83, 57, 32, 102, 108, 72, 17, -1,
    -1, -1};
static __constant__ signed char kA1Task125[128] = {
    124, 38, 84, 41, 50, 45, 43, 36, 14, 119, 24, 105, 35, 93, 59, 18, 4, 121, 82, 7, 16, 39, 22, 9, 86, 73,
    104, 107, 64, 21, 103, 70, 74, 20, 113, 79, 110, 78, 96, 61, 81, 11, 19, 68, 80, 101, 31, 54, 85, 51, 46,
    6, 94, 109, 52, 47, 25, 71, 76, 116, 56, 65, 23, 106, 33, 10, 30, 123, 88, 42, 117, 53, 28, 99, 112, 91,
    92, 67, 13, 98, 5, 66, 87, 118, 122, 37, 44, 27, 40, 89, 0, 55, 12, 111, 49, 62, 90, 58, 95, 1, 69, 34,
    115, 3, 100, 60, 120, 97, 108, 75, 26, 57, 2, 29, 114, 77, 48, 83, 63, 15, 32, 8, 102, 72, 17, -1, -1,
    -1};

template <int KIND, int N>
struct Stp3Cfg {
  static constexpr int M = Pde<KIND, 3>::M;
  static constexpr int NPC = N * N * N;
  static constexpr int NF = N * N;
  static constexpr int THREADS = ((NPC + 31) / 32) * 32;
  static constexpr int G = EDG_STP3_G(N) < N ? EDG_STP3_G(N) : N;   // time nodes per group
  static constexpr int ROW = NPC;                             // one (axis, time node, component) row of axes 1, 2
  static constexpr bool A0NAT = EDG_STP3_A0NAT != 0;
  static constexpr bool A1TAB = EDG_STP3_A1TAB != 0 && N == 5 && EDG_STP3_KMAP(N) && M == 5;
  static constexpr bool A1NAT = !A1TAB && A0NAT && EDG_STP3_A1NAT != 0;
  static constexpr int ROW0 = A0NAT ? (N == 5 ? 137 : NPC + ((NPC + 1) & 1)) : NPC;   // rows of axis 0
  // plane tasks for axes 1 + 2 in full iterations (see kPlaneTask)
  static constexpr bool PLANE = EDG_STP3_PLANE != 0 && A1TAB && G == N && M == N && A0NAT;
  static constexpr int ROW1 = A1TAB ? (PLANE ? NPC : 133) : (A1NAT ? ROW0 : NPC);   // rows of axis 1
  static constexpr int FBUF = G * M * (ROW0 + ROW1 + ROW);
  static constexpr int STAGE = (1 + 3) * M * NPC;             // epilogue staging [(1+d) M][NPC]
  static constexpr int SF = FBUF > STAGE ? FBUF : STAGE;
  static constexpr int OPS = 2 * N + 2;                        // c = K^-1 lift, sum_s B[r][s]
  static constexpr size_t BYTES = sizeof(double) * (OPS + SF + 2 * M * NPC);
  static constexpr int MINB = EDG_STP3_MINB(N);
};

template <int KIND, int N>
__global__ void __launch_bounds__(Stp3Cfg<KIND, N>::THREADS, Stp3Cfg<KIND, N>::MINB)
stp_picard3_kernel(const StpArgs A) {
  const TraceScope trace_scope(A.trace);
  using Cf = Stp3Cfg<KIND, N>;
  constexpr int DIM = 3;
  constexpr int M = Cf::M, NPC = Cf::NPC, NF = Cf::NF, THREADS = Cf::THREADS, G = Cf::G, ROW = Cf::ROW;
  constexpr int O = pen_off(N);   // this order's block in the constant-bank operator table

  extern __shared__ __align__(16) double smem[];
  double* sC = smem;                 // K^-1 lift
  double* sBs = sC + N;              // sum_s B[r][s]
  double* sF = smem + Cf::OPS;       // flux / derivative rows [a][g][k][ROW]
  double* sQ0 = sF + Cf::SF;         // initial state [2][M][NPC] (thread-private)
  __shared__ double sIh[DIM];

  const int tid = threadIdx.x;
  const int node = tid;
  const bool lane_ok = node < NPC;
  // idle lanes read (and never write) the last node's rows: the same address
  // as lane NPC - 1 of their warp (a broadcast; node 0's address shared a bank
  // with the warp's first lane and cost an extra wavefront per load)
  const int nd = lane_ok ? node : NPC - 1;
  const int i0 = nd / NF, i1 = (nd / N) % N, i2 = nd % N;
  // position of this node in axis a's row layout (axes 1, 2 pencil-contiguous)
  const int pos[DIM] = {Cf::A0NAT ? nd : N * (i1 * N + i2) + i0,
                        Cf::A1TAB ? nd : (Cf::A1NAT ? NF * i1 + N * i2 + i0 : N * (i0 * N + i2) + i1),
                        N * (i0 * N + i1) + i2};
  // row (a, g, k): axis-0 rows (stride ROW0), axis-1 rows (ROW1), axis-2 rows (ROW)
  constexpr int ROW0 = Cf::ROW0, ROW1 = Cf::ROW1;
  auto row = [&](int a, int g, int k) -> int {
    return a == 0 ? (g * M + k) * ROW0
                  : (a == 1 ? G * M * ROW0 + (g * M + k) * ROW1 : G * M * (ROW0 + ROW1) + (g * M + k) * ROW);
  };
  // pencil layouts: axes 0 / 1 natural (pencil p at p, element stride n^2), else n p + j
  auto nat = [&](int a) { return (a == 0 && Cf::A0NAT) || (a == 1 && Cf::A1NAT); };
  const double dt = *A.dt;
  const int nblocks = A.nwork;
  // pencil-phase map: one (component, pencil) per thread when they fill the CTA
  constexpr bool KMAP = EDG_STP3_KMAP(N) && M * NF <= THREADS && 2 * M * NF > THREADS;
  const bool pb_ok = tid < M * NF;
  const int pk = pb_ok ? tid / NF : 0, pp = pb_ok ? tid % NF : 0;   // (component, pencil) of the pencil phase
  // axis-1 task under A1TAB: component and natural offset 25 i0 + i2 of the pencil
  const int t1 = Cf::A1TAB ? (int)(Cf::PLANE ? kA1Task125 : kA1Task)[tid < 128 ? tid : 127] : 0;
  // plane task (g, k, i0) of this thread: row r = g M + k, plane i0
  const int tpl = Cf::PLANE ? (int)kPlaneTask[tid < 128 ? tid : 127] : -1;
  const int pl_r = tpl >= 0 ? tpl / N : 0, pl_p = tpl >= 0 ? tpl % N : 0;
  const int pk1 = Cf::A1TAB ? (t1 >= 0 ? t1 / NF : 0) : pk;
  const int po1 = Cf::A1TAB ? (t1 >= 0 ? NF * ((t1 % NF) / N) + t1 % N : 0) : 0;

  auto prefetch_q = [&](int b, int buf) {
    if (lane_ok && b < A.nwork) {
      const int c = A.cell_list ? __ldg(A.cell_list + b) : b;
      const double* src = A.q + (size_t)c * M * NPC + node;
      double* dst = sQ0 + buf * M * NPC + node;
#pragma unroll
      for (int k = 0; k < M; ++k) cp_async8(dst + k * NPC, src + k * NPC);
    }
  };
  int blk = blockIdx.x;
  if (blk < nblocks) prefetch_q(blk, 0);
  cp_async_commit();
  // isotropic uniform cells (one h on every axis): 1/h moves from the pencil
  // outputs (one multiply per derivative value) into the time coefficients
  // (one per time node and iteration) -- a reassociation within the fp64
  // tolerance, not a change of the scheme
  const bool iso = EDG_STP3_ISO && !A.edges_per_cell && A.edges[0] == A.edges[1] && A.edges[1] == A.edges[2];
  const double ihs = iso ? 1.0 / A.edges[0] : 1.0;
  for (int i = tid; i < N; i += THREADS) {
    sC[i] = A.basis[EDG_BASIS_KLIFT(N) + i];
    double bs = 0.0;
    for (int s = 0; s < N; ++s) bs += A.basis[EDG_BASIS_KINV(N) + i * N + s] * (-dt * A.basis[EDG_BASIS_W(N) + s]);
    sBs[i] = bs * ihs;
  }
  if (!A.edges_per_cell && tid < DIM) sIh[tid] = 1.0 / A.edges[tid];
  unsigned its_sum = 0u;

  for (int gi = 0; blk < nblocks; blk += gridDim.x, ++gi) {
    const int cell = A.cell_list ? __ldg(A.cell_list + blk) : blk;
    if (blk + (int)gridDim.x < nblocks) prefetch_q(blk + gridDim.x, (gi + 1) & 1);
    cp_async_commit();
    if (A.edges_per_cell && tid < DIM) sIh[tid] = 1.0 / A.edges[(size_t)cell * DIM + tid];
    cp_async_wait1();
    __syncthreads();   // operators, 1/h, flags (and the previous block's epilogue reads) settled

    const double* const q0s = sQ0 + (gi & 1) * M * NPC + node;
    double qh[N][M], acc[N][M];
#pragma unroll
    for (int k = 0; k < M; ++k) {
      const double v = lane_ok ? q0s[k * NPC] : 1.0;
#pragma unroll
      for (int r = 0; r < N; ++r) qh[r][k] = v;
    }

    // ---- phase helpers -------------------------------------------------
    // A: flux of time node s (group slot g) at this node -> rows [a][g][k]
    auto put_flux = [&](int g, const double* q) {
      double F[DIM][M];
      FastFlux<KIND, DIM>::template all<M>(q, A.pp, F);
      if (lane_ok) {
#pragma unroll
        for (int a = 0; a < DIM; ++a)
#pragma unroll
          for (int k = 0; k < M; ++k) sF[row(a, g, k) + pos[a]] = F[a][k];
      }
    };
    // B: in-place pencil contraction of the rows of group slots [0, ng)
    auto pencils = [&](int ng) {
      if constexpr (Cf::PLANE) {
        if (ng == G) {
          auto run = [&](auto scaled) {
            constexpr bool SC = decltype(scaled)::value;
            // axis 0: the thread's (component, pencil) in every time node's row
            if (pb_ok) {
              const double ih = SC ? sIh[0] : 1.0;
#pragma unroll
              for (int g = 0; g < G; ++g) {
                double* P = sF + row(0, g, pk) + pp;
                double f[N];
#pragma unroll
                for (int j = 0; j < N; ++j) f[j] = P[j * NF];
#pragma unroll
                for (int i = 0; i < N; ++i) {
                  double h = 0.0;
#pragma unroll
                  for (int j = 0; j < N; ++j) h = fma(kPen[O + EDG_BASIS_D(N) + i * N + j], f[j], h);
                  P[i * NF] = SC ? h * ih : h;
                }
              }
            }
            // axes 1 + 2: one plane task
            if (tpl >= 0) {
              const double ih1 = SC ? sIh[1] : 1.0, ih2 = SC ? sIh[2] : 1.0;
              const double* P1 = sF + G * M * ROW0 + pl_r * ROW1 + NF * pl_p;
              double* P2 = sF + G * M * (ROW0 + ROW1) + pl_r * ROW + NF * pl_p;
              double f1[N][N];
#pragma unroll
              for (int l = 0; l < N; ++l)
#pragma unroll
                for (int j = 0; j < N; ++j) f1[l][j] = P1[l * N + j];
#pragma unroll
              for (int i = 0; i < N; ++i) {
                double f2[N], o[N];
#pragma unroll
                for (int l = 0; l < N; ++l) f2[l] = P2[i * N + l];
#pragma unroll
                for (int j = 0; j < N; ++j) {
                  double h1 = 0.0, h2 = 0.0;
#pragma unroll
                  for (int l = 0; l < N; ++l) {
                    h1 = fma(kPen[O + EDG_BASIS_D(N) + i * N + l], f1[l][j], h1);
                    h2 = fma(kPen[O + EDG_BASIS_D(N) + j * N + l], f2[l], h2);
                  }
                  o[j] = SC ? fma(h1, ih1, h2 * ih2) : h1 + h2;
                }
#pragma unroll
                for (int j = 0; j < N; ++j) P2[i * N + j] = o[j];
              }
            }
          };
          if (iso)
            run(std::false_type{});
          else
            run(std::true_type{});
          return;
        }
      }
      if constexpr (KMAP) {
        // thread (component k, pencil p): every row (a, g, k) of its k at its
        // pencil -- no index arithmetic, and the warp-wide stride-n accesses
        // of two consecutive k rows (row stride n^3) stay at two wavefronts
        auto run = [&](auto scaled) {
#pragma unroll
          for (int a = 0; a < DIM; ++a) {
            const double ih = decltype(scaled)::value ? sIh[a] : 1.0;
#pragma unroll
            // pencil element j: axis 0 (natural rows) at p + n^2 j, else n p + j
            const bool tab = a == 1 && Cf::A1TAB;
            const int js = tab ? N : (nat(a) ? NF : 1);
            const int po = tab ? po1 : (nat(a) ? pp : pp * N);
            const int kk = tab ? pk1 : pk;
#pragma unroll
            for (int g = 0; g < G; ++g) {
              if (g < ng) {
                double* P = sF + row(a, g, kk) + po;
                double f[N];
#pragma unroll
                for (int j = 0; j < N; ++j) f[j] = P[j * js];
#pragma unroll
                for (int i = 0; i < N; ++i) {
                  double h = 0.0;
#pragma unroll
                  for (int j = 0; j < N; ++j) h = fma(kPen[O + EDG_BASIS_D(N) + i * N + j], f[j], h);
                  P[i * js] = decltype(scaled)::value ? h * ih : h;
                }
              }
            }
          }
        };
        if (pb_ok) {
          if (iso)
            run(std::false_type{});
          else
            run(std::true_type{});
        }
        return;
      }
      const int tasks = DIM * ng * M * NF;
      for (int t = tid; t < tasks; t += THREADS) {
        const int rg = t / NF, p = t - rg * NF;          // rg = (a, g, k) within the used slots
        const int a = rg / (ng * M), rem = rg - a * ng * M;
        const bool na = nat(a);
        const int js = na ? NF : 1;
        double* P = sF + row(a, rem / M, rem % M) + (na ? p : p * N);
        double f[N];
#pragma unroll
        for (int j = 0; j < N; ++j) f[j] = P[j * js];
        const double ih = iso ? 1.0 : sIh[a];
#pragma unroll
        for (int i = 0; i < N; ++i) {
          double h = 0.0;
#pragma unroll
          for (int j = 0; j < N; ++j) h = fma(kPen[O + EDG_BASIS_D(N) + i * N + j], f[j], h);
          P[i * js] = h * ih;
        }
      }
    };
    // C: divergence of group slot g at this node
    auto div_at = [&](int g, double (&dv)[M], bool plane = false) {
      if (Cf::PLANE && plane) {
        // axis 0 + the plane tasks' sum of axes 1 and 2 (left in axis 2's rows)
#pragma unroll
        for (int k = 0; k < M; ++k) dv[k] = sF[row(0, g, k) + pos[0]] + sF[row(2, g, k) + pos[2]];
        return;
      }
#pragma unroll
      for (int k = 0; k < M; ++k)
        dv[k] = (sF[row(0, g, k) + pos[0]] + sF[row(1, g, k) + pos[1]]) + sF[row(2, g, k) + pos[2]];
    };

    int its = 0;
    bool conv = false, inacc = false;
    const int max_iter = A.max_iter;
    // iteration exit (kernels.py:143-147): delta = max |new - qhat| < tol,
    // NaN never below -- "every |new - qhat| < tol" per thread, OR-reduced
    auto finish = [&](int it, bool below) -> bool {
      const bool any = __syncthreads_or(lane_ok && !below);
      its = it;
      if (!any) conv = true;
      return any;
    };
    bool any = false;
    if (max_iter >= 1) {
      // reduced first iteration: qhat_s = q for every s (kernels.py:134), so
      //   acc[r] = c_r q + (sum_s B[r][s]) div F(q)
      {
        double q[M];
#pragma unroll
        for (int k = 0; k < M; ++k) q[k] = qh[0][k];
        put_flux(0, q);
      }
      __syncthreads();
      pencils(1);
      __syncthreads();
      double dv[M];
      div_at(0, dv);
#pragma unroll
      for (int k = 0; k < M; ++k)
#pragma unroll
        for (int r = 0; r < N; ++r) acc[r][k] = fma(sBs[r], dv[k], sC[r] * qh[r][k]);
      bool below = true;
#pragma unroll
      for (int r = 0; r < N; ++r)
#pragma unroll
        for (int k = 0; k < M; ++k) below = below & (fabs(acc[r][k] - qh[r][k]) < A.tol);
      inacc = true;
      any = finish(1, below);
    }
    // full iteration: qn = c q + sum_s B[r][s] div F(qc_s); returns "not converged"
    auto body = [&](const double (&qc)[N][M], double (&qn)[N][M], int it) -> bool {
#pragma unroll
      for (int s0 = 0; s0 < N; s0 += G) {
        const int ng = (N - s0) < G ? (N - s0) : G;
#pragma unroll
        for (int g = 0; g < G; ++g)
          if (g < ng) {
            double q[M];
#pragma unroll
            for (int k = 0; k < M; ++k) q[k] = qc[s0 + g][k];
            put_flux(g, q);
          }
        __syncthreads();
        pencils(ng);
        __syncthreads();
        if (s0 == 0) {
          // the new iterate starts from the lift of the initial state (set
          // here, after the pencil / plane phase, so it is not live across it)
#pragma unroll
          for (int k = 0; k < M; ++k) {
            const double q0 = lane_ok ? q0s[k * NPC] : 1.0;
#pragma unroll
            for (int r = 0; r < N; ++r) qn[r][k] = kPen[O + EDG_BASIS_KLIFT(N) + r] * q0;
          }
        }
#pragma unroll
        for (int g = 0; g < G; ++g)
          if (g < ng) {
            double dv[M];
            div_at(g, dv, ng == G);
            const double sc = -(dt * kPen[O + EDG_BASIS_W(N) + s0 + g]) * ihs;   // (-dt) w_s (/ h when iso)
#pragma unroll
            for (int r = 0; r < N; ++r) {
              const double b = kPen[O + EDG_BASIS_KINV(N) + r * N + s0 + g] * sc;
#pragma unroll
              for (int k = 0; k < M; ++k) qn[r][k] = fma(b, dv[k], qn[r][k]);
            }
          }
        if (s0 + G < N) __syncthreads();   // the next group's fluxes overwrite the rows
      }
      bool below = true;
#pragma unroll
      for (int r = 0; r < N; ++r)
#pragma unroll
        for (int k = 0; k < M; ++k) below = below & (fabs(qn[r][k] - qc[r][k]) < A.tol);
      return finish(it, below);   // the barrier also guards the rows for the next iteration
    };
    // EDG_STP3_PP = 1: the loop is unrolled by two so that qh and acc swap roles
    // (no copies, but two copies of the iteration body in the instruction
    // stream); 0: one body, the new iterate copied back
#ifndef EDG_STP3_PP
#define EDG_STP3_PP 1
#endif
    if constexpr (EDG_STP3_PP != 0) {
      for (int it = 2; any && it <= max_iter;) {
        any = body(acc, qh, it);
        inacc = false;
        if (!any || ++it > max_iter) break;
        any = body(qh, acc, it);
        inacc = true;
        ++it;
      }
    } else {
#pragma unroll 1
      for (int it = 2; any && it <= max_iter; ++it) {
        any = body(acc, qh, it);
        inacc = false;
#pragma unroll
        for (int r = 0; r < N; ++r)
#pragma unroll
          for (int k = 0; k < M; ++k) acc[r][k] = qh[r][k];
      }
    }
    if (inacc) {
#pragma unroll
      for (int r = 0; r < N; ++r)
#pragma unroll
        for (int k = 0; k < M; ++k) qh[r][k] = acc[r][k];
    }

    // ---------------------------------------------------------- epilogue --
    // q_end = sum_r l_r(1) qhat_r; q_int = dt sum_r w_r qhat_r;
    // fint_a = dt sum_r w_r F_a(qhat_r)     (kernels.py:148-155)
    double* St = sF;
    double qe[M], qi[M], fi[DIM][M];
#pragma unroll
    for (int k = 0; k < M; ++k) qe[k] = qi[k] = 0.0;
#pragma unroll
    for (int a = 0; a < DIM; ++a)
#pragma unroll
      for (int k = 0; k < M; ++k) fi[a][k] = 0.0;
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
    if (lane_ok) {
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
    for (int task = tid; task < DIM * NF; task += THREADS) {
      constexpr int PER_FAM = 2 * DIM * M * NF;
      const size_t tbase = (size_t)cell * PER_FAM;
      const int a = task / NF, f = task - a * NF;
      const int st = a == DIM - 1 ? 1 : (a == 0 ? NF : N);
      const int hi = f / st, lo = f - hi * st;
      const int base = hi * st * N + lo;
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
    // (the next block's first barrier orders these staging reads before its
    // flux writes)
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
