// Space-time predictor (Picard) kernel -- replaces kernels.py:120-159.
//
// Mapping: one thread per spatial node, CPB cells per
// CTA (~100-128 threads, 3 CTAs -- and barrier domains -- per SM in 2-D, 2 in
// 3-D), persistent CTAs walking Picard-ordered work blocks with the next
// block's initial state prefetched by cp.async.  A thread keeps the whole
// time column of its node in registers (qhat[n_t][m] and the next iterate
// acc[n_t][m], swapping roles every iteration), so the K^-1 time contraction
// is thread-local (K^-1 from the constant bank); the per-axis derivative
// contractions read the flux of a time node from shared memory.  In 2-D
// (even n) a lane quad is a 2x2 node block and the flux buffers are
// block-major, so each quad asks for 2 words per load (one wavefront).
//
// Per Picard iteration and cell, with B[r][s] = K^-1[r][s] * (-dt w_s) and
// c = K^-1 lift (kernels.py:134-142):
//     acc[r] = c_r q + sum_s B[r][s] sum_a (D/h_a) (x)_a F_a(qhat_s)
// then the per-cell exit of kernels.py:143-147 (delta = max |acc - qhat| <
// tol, NaN never below) is decided as "every |acc - qhat| < tol" by a
// per-thread predicate and a per-cell shared flag.  Converged cells stop
// updating; the CTA runs until its last cell stops (the solver orders cells
// by their previous Picard count so that CTAs are homogeneous).  The
// epilogue (kernels.py:148-157) forms q_end, q_int and the time-integrated
// flux, stages them in shared memory and projects them onto the 2d faces.
#pragma once
#include "edg_common.cuh"

namespace edg {

struct StpArgs {
  const double* q;
  const int32_t* cell_list;
  int32_t nwork;
  const double* basis;
  const double* edges;
  int32_t edges_per_cell;
  const double* dt;
  double tol;
  int32_t max_iter;
  PdeParams pp;
  double* q_end;
  double* q_int;
  double* trace_q;
  double* trace_f;
  int32_t* iterations;
  uint8_t* converged;
  unsigned long long* iter_total;   // optional: += sum of per-cell iterations
  unsigned long long* trace;        // optional launch-trace slot (TraceScope)
  // grid policy: 0 = persistent CTAs at full occupancy; > 0 = persistent, at
  // most that many CTAs per SM; < 0 = one work block per CTA, so the CTAs
  // retire as they finish and launches on higher-priority streams get their
  // slots (the enclave predictor of the two-stream schedule)
  int32_t ctas_per_sm;
};

constexpr int stp_best_cpb(int npc, int target) {
  if (npc >= target) return 1;
  int best = 1;
  double best_eff = 0.0;
  for (int c = 1; c * npc <= target + target / 4; ++c) {
    const int thr = ((c * npc + 31) / 32) * 32;
    const double eff = double(c * npc) / double(thr);
    if (eff >= best_eff - 1e-9) {
      best = c;
      best_eff = eff;
    }
  }
  return best;
}

// Lane -> node map of the 3-D p = 4 kernel (one 125-node cell per 128-thread
// CTA), opt-in EDG_STP_PERM3: lane quads are 2x2 'plates' of nodes (warps
// 0-1: (j,k) plates; warps 2-3: (j,k), (i,k), (i,j) plates and the leftover
// lines), so that two of the three derivative loads of a quad ask for 2 words
// split 2+2 (tools/perm/plates3d.py generates and models it; -1 = idle lane).
// Measured 12 % slower on cfg3: with row-major flux storage the plates raise
// bank conflicts (LDS.64 2.51 wavefronts, STS.64 4.25, vs 2.32 / 2.0).
static __constant__ int kStpPerm3d5[128] = {
    0, 1, 5, 6, 2, 3, 7, 8, 10, 11, 15, 16, 12, 13, 17, 18, 25, 26, 30, 31, 27, 28, 32, 33, 35, 36, 40,
    41, 37, 38, 42, 43, 50, 51, 55, 56, 52, 53, 57, 58, 60, 61, 65, 66, 62, 63, 67, 68, 75, 76, 80, 81,
    77, 78, 82, 83, 85, 86, 90, 91, 87, 88, 92, 93, 100, 101, 105, 106, 102, 103, 107, 108, 110, 111,
    115, 116, 112, 113, 117, 118, 20, 21, 45, 46, 22, 23, 47, 48, 70, 71, 95, 96, 72, 73, 97, 98, 4, 9,
    29, 34, 14, 19, 39, 44, 54, 59, 79, 84, 64, 69, 89, 94, 120, 121, 122, 123, 104, 109, 114, 119, 24,
    49, 74, 99, 124, -1, -1, -1};

// constant-bank copy of the basis table head (D, w, tl, tr, K^-1, K^-1 lift)
// for N = 2..8 at offsets pen_off(N); one copy per instantiation unit, filled
// by the launchers (device-to-device copy in stream order before the kernel)
constexpr int pen_ops(int n) { return 2 * n * n + 4 * n; }
constexpr int pen_off(int n) { return n <= 2 ? 0 : pen_off(n - 1) + pen_ops(n - 1); }
constexpr int kPenTotal = pen_off(9);
static __constant__ double kPen[kPenTotal];

#ifndef EDG_STP_MAP3
#define EDG_STP_MAP3 0
#endif

template <int DIM, int N>
struct StpCfg {
  static constexpr int NPC = ipow(N, DIM);
  static constexpr int NF = ipow(N, DIM - 1);
  // 2-D: ~100-128 threads per CTA (cfg2: 3 cells = 108 nodes in 128 threads,
  // cfg5: 6 cells = 96 nodes), 3 CTAs per SM at 168 registers -- measured
  // faster than 5 cells in 192 threads x 2 CTAs (smaller barrier domains);
  // 3-D: one 125-node cell per 128 threads
#ifndef EDG_STP_TARGET
#define EDG_STP_TARGET 100
#endif
  static constexpr int TARGET = EDG_STP_TARGET;
  static constexpr int CPB = stp_best_cpb(NPC, TARGET);
  static constexpr int THREADS = ((CPB * NPC + 31) / 32) * 32;
  // resident CTAs per SM requested from ptxas (caps registers per thread)
  // (measured: 2 for the 2-D p=5 kernel; 2 for the 3-D p=4 kernel since the
  // constant-bank K^-1 and the unrolled Picard loop: 255 registers, 8 warps
  // per SM, 3 % faster than 3 CTAs at 168 registers)
#ifndef EDG_STP_MINB_3D
#define EDG_STP_MINB_3D 2
#endif
#ifndef EDG_STP_MINB_2D
#define EDG_STP_MINB_2D 3
#endif
  // 2-D n = 4 (cfg5's p = 3): its own cap (A/B: EDG_STP_MINB_2D_N4)
#ifndef EDG_STP_MINB_2D_N4
#define EDG_STP_MINB_2D_N4 5   // 128 registers, 5 CTAs per SM: cfg5 graph step 48.2 -> 46.4 us
#endif
  static constexpr int MINB = DIM == 2 ? (N == 4 ? EDG_STP_MINB_2D_N4 : EDG_STP_MINB_2D) : EDG_STP_MINB_3D;
};

template <int KIND, int DIM, int N>
struct StpSmem {
  using C = StpCfg<DIM, N>;
  static constexpr int M = Pde<KIND, DIM>::M;
  static constexpr int OPS = 2 * N * N + 6 * N;                 // D, B, w, tr, tl, c, Bsum (+pad)
  // flux buffers pad the last (contiguous) axis to an even length NP so that
  // pencil pairs along it are 16-byte aligned
  static constexpr int NP = N;   // (padding odd N to N+1 for pair loads measured slower on 3-D p=4)
  static constexpr int NPCP = C::NPC / N * NP;
  // EDG_STP_T0=1 (2-D, even N): store the axis-0 flux transposed ([k][j][i],
  // pencils contiguous) so both derivative axes use 16-byte pair loads
  // (measured 3% slower on cfg2 at CFL 0.9: off by default)
#ifndef EDG_STP_T0
#define EDG_STP_T0 0
#endif
  static constexpr bool T0 = EDG_STP_T0 && DIM == 2 && N % 2 == 0;
  // EDG_STP_SPAD=1: per-cell flux block stride padded (EDG_STP_SPAD_MOD mod
  // 16 doubles) so the same pencil of two cells sharing a warp lands on
  // different banks (without quads measured no faster: off by default)
#ifndef EDG_STP_SPAD
#define EDG_STP_SPAD 0
#endif
  // with lane quads a warp's 16 distinct words of one axis-0 load fill all
  // 32 banks only if the two cells of a warp are 16 banks apart
#ifndef EDG_STP_SPAD_QUAD
#define EDG_STP_SPAD_QUAD 1
#endif
  // two interleaved FMA chains per derivative dot product: measured +2 % on
  // 3-D p=4 and -5 % on 2-D p=5, so on by default in 3-D only
  // (EDG_STP_CH2=0/1 forces it)
#ifndef EDG_STP_CH2
#define EDG_STP_CH2 (-1)
#endif
  static constexpr bool CH2 = EDG_STP_CH2 < 0 ? DIM == 3 : EDG_STP_CH2 != 0;
  // EDG_STP_QUAD (default 1): 2x2-node lane quads on 2-D even-N cells
#ifndef EDG_STP_QUAD
#define EDG_STP_QUAD 1
#endif
  static constexpr bool QUAD = EDG_STP_QUAD && DIM == 2 && N % 2 == 0 && !T0;
  // EDG_STP_BM (default 1, with QUAD): flux buffers in 2x2-block-major node
  // order (the lane order), so a warp's flux stores are 32 consecutive words
  // (bank-conflict-free) and a quad's two words of a load are adjacent
#ifndef EDG_STP_BM
#define EDG_STP_BM 1
#endif
  static constexpr bool BM = QUAD && EDG_STP_BM;
  static constexpr int SS0 = DIM * M * NPCP;
  static constexpr bool SPADX = (EDG_STP_SPAD || (QUAD && EDG_STP_SPAD_QUAD)) && C::CPB > 1;
  // cell stride mod 16 doubles.  A quad's axis-0 load asks for 2 adjacent
  // doubles at (c/2) 4 + const, i.e. double banks {0,1}, {4,5}, {8,9} for the
  // three quad columns of a cell; a second cell sharing the warp lands on the
  // free banks iff its block starts at 2, 6, 10 or 14 (mod 16).  Measured on
  // cfg2 (CFL 0.9, steps 1-10): 8 -> 0.649 ms, 2 -> 0.626, 4 -> 0.626,
  // 14 -> 0.629; indifferent on cfg5
#ifndef EDG_STP_SPAD_MOD
#define EDG_STP_SPAD_MOD 2
#endif
  static constexpr int SS = SPADX ? SS0 + ((EDG_STP_SPAD_MOD - SS0 % 16) + 16) % 16 : SS0;
  static constexpr int FB = C::CPB * SS;                        // one flux buffer
  // time nodes per pipeline stage (one barrier per stage); EDG_STP_G overrides
#if defined(EDG_STP_G)
  static constexpr int G = EDG_STP_G;
#else
#ifndef EDG_STP_G2D
#define EDG_STP_G2D 2
#endif
#ifndef EDG_STP_G3D
#define EDG_STP_G3D 2
#endif
  // 2-D n >= 6: all time nodes in one stage (one flux barrier per iteration;
  // +1.5 % on cfg2), smaller n: pipelined pairs (+6 % on cfg5's n = 4)
#ifndef EDG_STP_G2D_BIG
#define EDG_STP_G2D_BIG 8
#endif
  // 3-D: pipelined pairs (one stage of all 5 time nodes measured +1 % over
  // steps 4-9 of cfg3 but 31 % slower over the full 20-step bench)
#ifndef EDG_STP_G3D_BIG
#define EDG_STP_G3D_BIG 2
#endif
  static constexpr int G = DIM == 2 ? (N >= 6 ? EDG_STP_G2D_BIG : EDG_STP_G2D) : (N <= 5 ? EDG_STP_G3D_BIG : EDG_STP_G3D);
#endif
  // EDG_STP_QHS: keep the Picard iterate qhat in (thread-private) shared
  // memory instead of registers (fewer registers, more resident CTAs)
#ifdef EDG_STP_QHS
  static constexpr bool QHS = true;
#else
  static constexpr bool QHS = false;
#endif
  static constexpr int QH = QHS ? C::CPB * N * M * C::NPC : 0;
  // EDG_STP_PP (default 1): unroll the Picard loop by two so that qhat and
  // the next iterate swap register roles instead of being copied
#ifndef EDG_STP_PP
#define EDG_STP_PP 1
#endif
  static constexpr bool PP = EDG_STP_PP && !QHS;
  // EDG_STP_KC (default 1): the time contraction takes K^-1 from the constant
  // bank (kPen, an FMA operand: no shared load) and scales the derivative by
  // (-dt) w_s first -- the reference's own order (kernels.py:141-142)
  // KC = 1 scales the derivative, KC = 2 scales K^-1 per (r, s) (B bit-identical
  // to the shared-memory table); measured best: 2 (+8 % on cfg2 at CFL 0.9;
  // on the full 20-step cfg3 bench 2 beats 1 by 0.4 % and 0 by 1.1 %)
#ifndef EDG_STP_KC
#define EDG_STP_KC (-1)
#endif
  static constexpr int KCM = EDG_STP_KC < 0 ? 2 : EDG_STP_KC;
  static constexpr bool KC = KCM != 0 && PP;
  // flux stages: double-buffered groups of G time nodes, or one stage holding
  // all time nodes when G >= N
  static constexpr int STAGES = G >= N ? 1 : 2;
  static constexpr size_t BYTES = sizeof(double) * (OPS + STAGES * G * FB + 2 * C::CPB * M * C::NPC + QH) + sizeof(int) * 2 * C::CPB;
};

template <int KIND, int DIM, int N, int MINB = StpCfg<DIM, N>::MINB>
__global__ void __launch_bounds__(StpCfg<DIM, N>::THREADS, MINB)
stp_picard_kernel(const StpArgs A) {
  const TraceScope trace_scope(A.trace);
  using P = Pde<KIND, DIM>;
  using Cf = StpCfg<DIM, N>;
  using Sm = StpSmem<KIND, DIM, N>;
  constexpr int M = P::M;
  constexpr int NPC = Cf::NPC;
  constexpr int NF = Cf::NF;
  constexpr int CPB = Cf::CPB;
  constexpr int THREADS = Cf::THREADS;
  // flux buffer layout: component-major [a][k][node] (a node-major variant with
  // 16-byte accesses measured slower: 2-way bank conflicts from the node stride)

  extern __shared__ __align__(16) double smem[];
  double* sD = smem;                 // D[N][N]
  double* sB = sD + N * N;           // B[r][s]
  double* sW = sB + N * N;
  double* sTL = sW + N;
  double* sTR = sTL + N;
  double* sC = sTR + N;              // K^-1 lift
  double* sBs = sC + N;              // sum_s B[r][s]
  double* sF = smem + Sm::OPS;       // flux buffers [2][CPB][DIM][M][NPCP], 16-byte aligned (OPS even)
  static_assert(Sm::OPS % 2 == 0 && Sm::OPS >= 2 * N * N + 5 * N, "operator block must keep sF 16-byte aligned");
  double* sQ0 = sF + Sm::STAGES * Sm::G * Sm::FB;                       // initial state [2][CPB][M][NPC] (thread-private)
  double* sQH = sQ0 + 2 * CPB * M * NPC;                      // qhat [CPB][N][M][NPC] when Sm::QHS
  int* sFlag = reinterpret_cast<int*>(sQH + Sm::QH);          // [2][CPB] "not converged" flags

  const int tid = threadIdx.x;
  int slot, node;
  bool lane_ok;
  // EDG_STP_PERM3=1: the 2x2-plate lane map of tools/perm/plates3d.py
#ifndef EDG_STP_PERM3
#define EDG_STP_PERM3 0
#endif
  constexpr bool kUsePerm3d5 = EDG_STP_PERM3 != 0;
  if constexpr (kUsePerm3d5 && DIM == 3 && N == 5 && CPB == 1) {
    // compact lane->node blocks: <= 16 distinct pencils per warp on most axes
    const int v = kStpPerm3d5[tid];
    slot = 0;
    node = v < 0 ? 0 : v;
    lane_ok = v >= 0;
  } else if constexpr (Sm::QUAD) {
    // 2-D, even N: lane quad (4 consecutive lanes) = one 2x2 block of nodes,
    // so every derivative load of a quad touches 2 distinct words (2 rows on
    // axis 1, 2 columns on axis 0) -- one wavefront per warp-wide LDS.64
    // instead of two (measured: a quad is served <= 2 distinct addresses per
    // wavefront)
    constexpr int HB = N / 2, QPC = HB * HB;
    const int qd = tid >> 2, u = tid & 3;
    slot = qd / QPC;
    const int b = qd - slot * QPC;
    node = (2 * (b / HB) + (u >> 1)) * N + 2 * (b % HB) + (u & 1);
    lane_ok = slot < CPB;
  } else if constexpr (DIM == 3 && CPB == 1 && EDG_STP_MAP3 != 0) {
    // EDG_STP_MAP3 = 1: lanes run fastest along axis 0 (node (i, j, k) at lane
    // (j n + k) n + i); = 2: fastest along axis 1 (lane (i n + k) n + j)
    slot = tid / NPC;
    const int t = tid - slot * NPC;
    const int f = t % N, p = t / N;
    node = EDG_STP_MAP3 == 1 ? f * N * N + p : (p / N) * N * N + f * N + p % N;
    lane_ok = slot < CPB;
  } else {
    slot = tid / NPC;
    node = tid - slot * NPC;
    lane_ok = slot < CPB;
  }
  const double dt = *A.dt;
  // persistent CTAs: work blocks blockIdx.x, blockIdx.x + gridDim.x, ...; the
  // next block's initial state is copied into the other staging buffer with
  // cp.async while this one iterates (thread-private: each thread copies and
  // later reads only its own node, so no barrier guards the buffers)
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

  for (int i = tid; i < N * N; i += THREADS) {
    sD[i] = A.basis[EDG_BASIS_D(N) + i];
    const int s = i % N;
    // B[r][s] = K^-1[r][s] * ((-dt) * w[s])   (kernels.py:141-142 folded)
    sB[i] = A.basis[EDG_BASIS_KINV(N) + i] * (-dt * A.basis[EDG_BASIS_W(N) + s]);
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
  // pencil base (node index with i_a = 0) per axis
  constexpr int NP = Sm::NP, NPCP = Sm::NPCP;
  const int bnode = (node / N) * NP + node % N;   // node index in the padded flux buffer
  int pb[DIM];
#pragma unroll
  for (int a = 0; a < DIM; ++a) pb[a] = bnode - ix[a] * (a == DIM - 1 ? 1 : NP * ipow(N, DIM - 2 - a));
  // transposed axis-0 layout: node (i, j) stored at j * N + i, pencil base j * N
  const int tnode = DIM == 2 ? ix[DIM - 1] * N + ix[0] : 0;
  if constexpr (Sm::T0) pb[0] = ix[DIM - 1] * N;
  // block-major flux layout: node (r, c) at ((r/2) HB + c/2) 4 + (r%2) 2 + c%2
  constexpr int HB2 = N / 2;
  auto bpos = [&](int r, int c) { return ((r >> 1) * HB2 + (c >> 1)) * 4 + (r & 1) * 2 + (c & 1); };
  const int fnode = Sm::BM ? bpos(ix[0], ix[DIM - 1]) : bnode;
  if constexpr (Sm::BM) {
    pb[0] = bpos(0, ix[DIM - 1]);
    pb[DIM - 1] = bpos(ix[0], 0);
  }
  // offset of the j-th node of a pencil along axis a from its base pb[a]
  auto fofs = [&](int a, int j, int st) {
    if constexpr (Sm::BM) return a == 0 ? (j >> 1) * HB2 * 4 + (j & 1) * 2 : (j >> 1) * 4 + (j & 1);
    else return (a == DIM - 1 || (Sm::T0 && a == 0)) ? j : j * st;
  };
  unsigned its_sum = 0u;
#ifndef EDG_STP_CLIFT
#define EDG_STP_CLIFT 1
#endif
#ifndef EDG_STP_IHS
#define EDG_STP_IHS 1
#endif
#ifndef EDG_STP_DRH
#define EDG_STP_DRH 1
#endif
  // derivative rows of this node, scaled by 1/h_a: once per CTA on uniform
  // meshes (shared edges), per work block when the edges are per cell
  double Dr[DIM][N];
  // uniform meshes: 1/h_a once per CTA in shared memory (the per-block
  // rebuild of the 2-D rows then costs no division and no global load)
  __shared__ double sIh[DIM];
  if (!A.edges_per_cell && tid < DIM) sIh[tid] = 1.0 / A.edges[tid];
  __syncthreads();
  auto load_dr = [&](int cell) {
    const double* e = A.edges + (A.edges_per_cell ? (size_t)cell * DIM : 0);
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
      const double ih = (EDG_STP_IHS && !A.edges_per_cell) ? sIh[a] : 1.0 / e[a];
#pragma unroll
      for (int j = 0; j < N; ++j) Dr[a][j] = sD[ix[a] * N + j] * ih;
    }
  };
  constexpr bool kDrOnce = EDG_STP_DRH != 0 && DIM == 3;   // (2-D n = 6: spills at the 3-CTA cap)
  if (kDrOnce && !A.edges_per_cell) load_dr(0);

  for (int gi = 0; blk < nblocks; blk += gridDim.x, ++gi) {
  const int item = blk * CPB + slot;
  const bool has_cell = lane_ok && (item < A.nwork);
  const int cell = has_cell ? (A.cell_list ? __ldg(A.cell_list + item) : item) : 0;
  if (blk + (int)gridDim.x < nblocks) prefetch_q(blk + gridDim.x, (gi + 1) & 1);
  cp_async_commit();
  if (tid < 2 * CPB) sFlag[tid] = 0;
  if (!kDrOnce || A.edges_per_cell) load_dr(cell);
  cp_async_wait1();   // this block's initial state (own node) has landed

  // the initial state is re-read every iteration (c_r q): private copy in
  // shared memory
  double* const q0s = sQ0 + (gi & 1) * QB + slot * M * NPC + node;
  constexpr bool QHS = Sm::QHS;
  double qhr[QHS ? 1 : N][M], acc[N][M];
  double* const qhs = sQH + slot * N * M * NPC + node;
  auto qget = [&](int r, int k) -> double {
    if constexpr (QHS) return qhs[(r * M + k) * NPC];
    else return qhr[r][k];
  };
  auto qset = [&](int r, int k, double v) {
    if constexpr (QHS) {
      if (lane_ok) qhs[(r * M + k) * NPC] = v;
    } else {
      qhr[r][k] = v;
    }
  };
  auto qrow = [&](int r, double (&out)[M]) {
#pragma unroll
    for (int k = 0; k < M; ++k) out[k] = qget(r, k);
  };
#pragma unroll
  for (int k = 0; k < M; ++k) {
    const double v = has_cell ? q0s[k * NPC] : 1.0;
#pragma unroll
    for (int r = 0; r < N; ++r) qset(r, k, v);
  }

  bool active = has_cell;
  int its = 0;
  bool conv = false;
  const int max_iter = A.max_iter;
  double* const buf0 = sF + slot * Sm::SS;
  double* const buf1 = buf0 + Sm::FB;

  // flux of one time node of this node's column -> flux buffer [a][k][node]
  auto put_flux = [&](double* Fb, const double* q) {
    double F[DIM][M];
    FastFlux<KIND, DIM>::template all<M>(q, A.pp, F);
#pragma unroll
    for (int a = 0; a < DIM; ++a)
#pragma unroll
      for (int k = 0; k < M; ++k) Fb[(a * M + k) * NPCP + ((Sm::T0 && a == 0) ? tnode : fnode)] = F[a][k];
  };
  // dv[k] = sum_a sum_j (D/h_a)[i_a][j] F_a[k][pencil_a(j)]
  auto deriv = [&](const double* Fb, double (&dv)[M]) {
    // 2-D: one independent FMA chain per (axis, component) for ILP, summed at
    // the end; 3-D: one chain per component (measured faster: fewer registers)
    constexpr bool SPLIT = DIM == 2;
    double part[DIM][M];
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
      const int st = a == DIM - 1 ? 1 : NP * ipow(N, DIM - 2 - a);
#pragma unroll
      for (int k = 0; k < M; ++k) {
        const double* Fa = Fb + (a * M + k) * NPCP + pb[a];
        double acc_ak = (SPLIT || a == 0) ? 0.0 : part[a > 0 ? a - 1 : 0][k];
        if ((a == DIM - 1 || (Sm::T0 && a == 0)) && (N % 2 == 0)) {
          // contiguous pencil: 16-byte pair loads (lanes of one pencil broadcast)
#pragma unroll
          if constexpr (Sm::CH2) {
            // two interleaved chains (even / odd j): half the dependent-FMA depth
            double acc_b = 0.0;
#pragma unroll
            for (int j = 0; j + 1 < N; j += 2) {
              const double2 v = *reinterpret_cast<const double2*>(Fa + fofs(a, j, st));
              acc_ak = fma(Dr[a][j], v.x, acc_ak);
              acc_b = fma(Dr[a][j + 1], v.y, acc_b);
            }
            if (N & 1) acc_ak = fma(Dr[a][N - 1], Fa[fofs(a, N - 1, st)], acc_ak);
            acc_ak += acc_b;
          } else {
#pragma unroll
            for (int j = 0; j + 1 < N; j += 2) {
              const double2 v = *reinterpret_cast<const double2*>(Fa + fofs(a, j, st));
              acc_ak = fma(Dr[a][j], v.x, acc_ak);
              acc_ak = fma(Dr[a][j + 1], v.y, acc_ak);
            }
            if (N & 1) acc_ak = fma(Dr[a][N - 1], Fa[fofs(a, N - 1, st)], acc_ak);
          }
        } else if constexpr (Sm::CH2) {
          double acc_b = 0.0;
#pragma unroll
          for (int j = 0; j < N; ++j) {
            if (j & 1) acc_b = fma(Dr[a][j], Fa[fofs(a, j, st)], acc_b);
            else acc_ak = fma(Dr[a][j], Fa[fofs(a, j, st)], acc_ak);
          }
          acc_ak += acc_b;
        } else {
#pragma unroll
          for (int j = 0; j < N; ++j) acc_ak = fma(Dr[a][j], Fa[fofs(a, j, st)], acc_ak);
        }
        part[a][k] = acc_ak;
      }
    }
#pragma unroll
    for (int k = 0; k < M; ++k) {
      if (SPLIT) {
        double v = part[0][k];
#pragma unroll
        for (int a = 1; a < DIM; ++a) v += part[a][k];
        dv[k] = v;
      } else {
        dv[k] = part[DIM - 1][k];
      }
    }
  };

  if constexpr (Sm::PP) {
    // ping-pong: odd iterations write acc, even ones qhr (no copies); the
    // latest iterate of this lane's cell is in acc iff inacc
    bool inacc = false;
    auto rowof = [&](const double (&qa)[N][M], int r, double (&out)[M]) {
#pragma unroll
      for (int k = 0; k < M; ++k) out[k] = qa[r][k];
    };
    // convergence flags and the CTA-wide continue decision (see below)
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
    auto body = [&](const double (&qc)[N][M], double (&qn)[N][M], int it, bool into_acc) -> bool {
        // G time nodes per barrier; stage buffers [2][G]
        constexpr int G = Sm::G;
        auto slotbuf = [&](int stage, int g) { return buf0 + (stage * G + g) * Sm::FB; };
        if (active) {
#pragma unroll
          for (int k = 0; k < M; ++k) {
            const double q0 = q0s[k * NPC];
#pragma unroll
            for (int r = 0; r < N; ++r) {
              // K^-1 lift: a uniform constant-bank operand when the table is there
              const double c = (Sm::KC && EDG_STP_CLIFT && DIM == 3) ? kPen[pen_off(N) + EDG_BASIS_KLIFT(N) + r] : sC[r];
              qn[r][k] = c * q0;
            }
          }
#pragma unroll
          for (int g = 0; g < G; ++g)
            if (g < N) {
              double q[M];
              rowof(qc, g, q);
              put_flux(slotbuf(0, g), q);
            }
        }
        __syncthreads();
        // software pipeline: the fluxes of the next G time nodes are evaluated
        // and stored (other stage) while the derivatives of this group are
        // contracted; one barrier per group
#pragma unroll
        for (int s0 = 0; s0 < N; s0 += G) {
          const int stage = (s0 / G) & 1;
          if (active) {
#pragma unroll
            for (int g = 0; g < G; ++g)
              if (s0 + G + g < N) {
                double q[M];
                rowof(qc, s0 + G + g, q);
                put_flux(slotbuf(stage ^ 1, g), q);
              }
#pragma unroll
            for (int g = 0; g < G; ++g) {
              if (s0 + g < N) {
                double dv[M];
                deriv(slotbuf(stage, g), dv);
                if constexpr (Sm::KC) {
                  constexpr int O = pen_off(N);
                  const double sc = -(dt * kPen[O + EDG_BASIS_W(N) + s0 + g]);   // = (-dt) w_s exactly
                  if constexpr (Sm::KCM == 1) {
#pragma unroll
                    for (int k = 0; k < M; ++k) dv[k] *= sc;
                  }
#pragma unroll
                  for (int r = 0; r < N; ++r) {
                    // KC = 2: B[r][s] = K^-1[r][s] * ((-dt) w_s), bit-identical to sB
                    const double b = Sm::KCM == 1 ? kPen[O + EDG_BASIS_KINV(N) + r * N + s0 + g]
                                                     : kPen[O + EDG_BASIS_KINV(N) + r * N + s0 + g] * sc;
#pragma unroll
                    for (int k = 0; k < M; ++k) qn[r][k] = fma(b, dv[k], qn[r][k]);
                  }
                } else {
#pragma unroll
                  for (int r = 0; r < N; ++r) {
                    const double b = sB[r * N + s0 + g];
#pragma unroll
                    for (int k = 0; k < M; ++k) qn[r][k] = fma(b, dv[k], qn[r][k]);
                  }
                }
              }
            }
          }
          __syncthreads();
        }
      bool below = true;
      if (active) {
#pragma unroll
        for (int r = 0; r < N; ++r)
#pragma unroll
          for (int k = 0; k < M; ++k) below = below & (fabs(qn[r][k] - qc[r][k]) < A.tol);
      }
      return finish(it, below, into_acc);
    };
    bool any = false;
    if (max_iter >= 1) {
        // qhat_s = q for every time node (kernels.py:134), so the first
        // iteration needs one flux and one derivative:
        //   acc[r] = c_r q + (sum_s B[r][s]) div F(q)
        if (active) {
          double q[M];
          qrow(0, q);
          put_flux(buf0, q);
        }
        __syncthreads();
        if (active) {
          double dv[M];
          deriv(buf0, dv);
#pragma unroll
          for (int k = 0; k < M; ++k) {
#pragma unroll
            for (int r = 0; r < N; ++r) acc[r][k] = fma(sBs[r], dv[k], sC[r] * qget(r, k));
          }
        }
      bool below = true;
      if (active) {
#pragma unroll
        for (int r = 0; r < N; ++r)
#pragma unroll
          for (int k = 0; k < M; ++k) below = below & (fabs(acc[r][k] - qhr[r][k]) < A.tol);
      }
      any = finish(1, below, true);
    }
    for (int it = 2; any && it <= max_iter;) {
      any = body(acc, qhr, it, false);
      if (!any || ++it > max_iter) break;
      any = body(qhr, acc, it, true);
      ++it;
    }
    if (inacc) {
#pragma unroll
      for (int r = 0; r < N; ++r)
#pragma unroll
        for (int k = 0; k < M; ++k) qhr[r][k] = acc[r][k];
    }
  } else {
    for (int it = 1; it <= max_iter; ++it) {
      if (it == 1) {
        // qhat_s = q for every time node (kernels.py:134), so the first
        // iteration needs one flux and one derivative:
        //   acc[r] = c_r q + (sum_s B[r][s]) div F(q)
        if (active) {
          double q[M];
          qrow(0, q);
          put_flux(buf0, q);
        }
        __syncthreads();
        if (active) {
          double dv[M];
          deriv(buf0, dv);
#pragma unroll
          for (int k = 0; k < M; ++k) {
#pragma unroll
            for (int r = 0; r < N; ++r) acc[r][k] = fma(sBs[r], dv[k], sC[r] * qget(r, k));
          }
        }
      } else {
        // G time nodes per barrier; stage buffers [2][G]
        constexpr int G = Sm::G;
        auto slotbuf = [&](int stage, int g) { return buf0 + (stage * G + g) * Sm::FB; };
        if (active) {
#pragma unroll
          for (int k = 0; k < M; ++k) {
            const double q0 = q0s[k * NPC];
#pragma unroll
            for (int r = 0; r < N; ++r) acc[r][k] = sC[r] * q0;
          }
#pragma unroll
          for (int g = 0; g < G; ++g)
            if (g < N) {
              double q[M];
              qrow(g, q);
              put_flux(slotbuf(0, g), q);
            }
        }
        __syncthreads();
        // software pipeline: the fluxes of the next G time nodes are evaluated
        // and stored (other stage) while the derivatives of this group are
        // contracted; one barrier per group
#pragma unroll
        for (int s0 = 0; s0 < N; s0 += G) {
          const int stage = (s0 / G) & 1;
          if (active) {
#pragma unroll
            for (int g = 0; g < G; ++g)
              if (s0 + G + g < N) {
                double q[M];
                qrow(s0 + G + g, q);
                put_flux(slotbuf(stage ^ 1, g), q);
              }
#pragma unroll
            for (int g = 0; g < G; ++g) {
              if (s0 + g < N) {
                double dv[M];
                deriv(slotbuf(stage, g), dv);
#pragma unroll
                for (int r = 0; r < N; ++r) {
                  const double b = sB[r * N + s0 + g];
#pragma unroll
                  for (int k = 0; k < M; ++k) acc[r][k] = fma(b, dv[k], acc[r][k]);
                }
              }
            }
          }
          __syncthreads();
        }
      }
      // delta = max |acc - qhat| < tol  <=>  every |acc - qhat| < tol (a NaN
      // fails the comparison exactly as it poisons np.max): a per-thread
      // predicate (DADD + DSETP.AND per value) and a per-cell "some lane is not
      // below tol" flag replace the max reduction
      int* flag = sFlag + (it & 1) * CPB;
      bool below = true;
      if (active) {
#pragma unroll
        for (int r = 0; r < N; ++r)
#pragma unroll
          for (int k = 0; k < M; ++k) {
            below = below & (fabs(acc[r][k] - qget(r, k)) < A.tol);
            qset(r, k, acc[r][k]);
          }
        if (!below) flag[slot] = 1;
      }
      // one barrier: the flags become visible, and the CTA goes on iff some
      // active cell has a lane not below tol (that cell stays active)
      const bool any = __syncthreads_or(active && !below);
      if (active) {
        its = it;
        if (flag[slot] == 0) {
          active = false;
          conv = true;
        }
      }
      // the other parity was last read before this barrier and is next written
      // after the next iteration's first barrier
      if (tid < CPB) sFlag[((it + 1) & 1) * CPB + tid] = 0;
      if (!any) break;
    }
  }

  // ---------------------------------------------------------- epilogue --
  // q_end = sum_r l_r(1) qhat_r; q_int = dt sum_r w_r qhat_r;
  // fint_a = dt sum_r w_r F_a(qhat_r)          (kernels.py:148-155)
  // staged as [slot][(1+DIM)*M][NPC] for the face projections
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
      const double tr = sTR[r], w = sW[r];
      double F[DIM][M];
      double q[M];
      qrow(r, q);
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
  // the flux buffers may still be read by other cells' last iteration until here
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
  // face projections, one task per (axis a, pencil f): the thread loads the
  // pencil of q_int and of fint_a once and writes both sides of both families
  // (trace_q / trace_f (a, 0) and (a, 1)) for all components
  constexpr int TASKS = DIM * NF;
  for (int task = node; has_cell && task < TASKS; task += NPC) {
    constexpr int PER_FAM = 2 * DIM * M * NF;
    const size_t tbase = (size_t)cell * PER_FAM;
    const int a = task / NF, f = task - a * NF;
    const int st = a == DIM - 1 ? 1 : ipow(N, DIM - 1 - a);
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
  if (has_cell && node == 0) its_sum += (unsigned)its;
  // staging / flux buffers are reused by the next work block
  __syncthreads();
  }  // work blocks
  if (A.iter_total) {
    // per-CTA sum of iteration counts (algorithmic-flop accounting), one atomic per CTA
    __shared__ unsigned int sIts;
    if (tid == 0) sIts = 0u;
    __syncthreads();
    if (its_sum) atomicAdd(&sIts, its_sum);
    __syncthreads();
    if (tid == 0 && sIts) atomicAdd(A.iter_total, (unsigned long long)sIts);
  }
}

}  // namespace edg
