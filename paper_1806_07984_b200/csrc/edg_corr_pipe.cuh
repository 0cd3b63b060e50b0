// Pipelined corrector for uniform Cartesian meshes (edg_corrector_grid) --
// the same computation and bits as corrector_kernel<..., FUSED = true> in
// edg_faces.cuh (kernels.py:162-193 + the admissible-dt candidate of
// kernels.py:267-281), restructured for HBM streaming:
//
//  * persistent CTAs (grid = SMs x resident CTAs) walk groups of CPB
//    consecutive cells;
//  * the next group's q_end block, own trace_q / trace_f blocks and the 2d
//    neighbour face traces are copied global -> shared with cp.async
//    (LDGSTS, 16-byte where aligned) while the current group is corrected
//    out of shared memory (two stages), so every SM always has a group's
//    bytes in flight instead of stalling each CTA on its own loads;
//  * the admissible-dt candidate and the non-finite count are reduced per
//    CTA across all its groups: one global atomic each per CTA.
#pragma once
#include "edg_faces.cuh"

namespace edg {

template <int KIND, int DIM, int N, bool GRID = true>
struct CorrPipe {
  using Cf = CorrCfg<DIM, N>;
  static constexpr int M = Pde<KIND, DIM>::M;
  static constexpr int NPC = Cf::NPC, NF = Cf::NF;
  // cells per group: the classic kernel's count, except one cell per group
  // when a cell already fills most of a 128-thread CTA (3-D p=4: 125 nodes),
  // so that two stages of the larger 3-D blocks still leave 4 CTAs per SM
#ifndef EDG_CORR_PIPE_TARGET
#define EDG_CORR_PIPE_TARGET 256
#endif
#ifndef EDG_CORR_CPB_BIG
#define EDG_CORR_CPB_BIG 1
#endif
  static constexpr int CPB = NPC >= 96 ? EDG_CORR_CPB_BIG : (EDG_CORR_PIPE_TARGET / NPC > 0 ? EDG_CORR_PIPE_TARGET / NPC : 1);
  // EDG_CORR_WIDE = 1: with one cell per group and more face points than
  // nodes (3-D p = 4: 150 > 125), the CTA is sized for the face points (one
  // Rusanov pass over 160 threads instead of two over 128).  Off by default
  // since q_end is loaded into registers: cfg3 1.50 ms at 128 threads against
  // 1.61 ms at 160
#ifndef EDG_CORR_WIDE
#define EDG_CORR_WIDE 0
#endif
  static constexpr int TOTF = 2 * DIM * NF;
  static constexpr bool WIDE = EDG_CORR_WIDE && CPB == 1 && TOTF > NPC;
  static constexpr int WORK = WIDE ? TOTF : CPB * NPC;
  static constexpr int THREADS = ((WORK + 31) / 32) * 32 < 64 ? 64 : ((WORK + 31) / 32) * 32;
  static constexpr int TRC = 2 * DIM * M * NF;            // trace doubles per cell (one family)
  // EDG_CORR_QEG (uniform grids, one cell per group): q_end is not staged --
  // each thread loads its node's values straight into registers at the start
  // of the group (5 KB less shared memory per stage on 3-D p = 4)
#ifndef EDG_CORR_QEG
#define EDG_CORR_QEG 1
#endif
  static constexpr bool QEG = EDG_CORR_QEG && GRID && CPB == 1;
  static constexpr int QE = QEG ? 0 : (CPB * M * NPC + 1) & ~1;     // stage sub-blocks, even -> 16-byte aligned
  static constexpr int TB = (CPB * TRC + 1) & ~1;
  // grid: q_end, trace_q, trace_f, neighbour trace_q;  adaptive: q_end,
  // trace_f, face outcomes (gathered through side_face)
  static constexpr int NB = GRID ? 3 : 2;
  static constexpr int STAGE = QE + NB * TB;
  static constexpr int NV = GRID ? 2 * DIM * N : CPB * 2 * DIM * N;    // lift vectors (per cell when adaptive)
  // resident CTAs asked of ptxas: 5 fit the shared memory of the unstaged-q_end 3-D kernel
  // 2-D: four CTAs per SM (64 registers) -- with ptxas's free choice (96
  // registers, 2 CTAs) the CTAs spun on the stage mbarrier (ncu: 40 % of the
  // samples on the wait loop's branch); cfg2 corrector 82.7 -> 66.0 (3) ->
  // 63.7 us (4)
#ifndef EDG_CORR_MINB_2D
#define EDG_CORR_MINB_2D 4
#endif
#ifndef EDG_CORR_MINB_3D
#define EDG_CORR_MINB_3D 5
#endif
  static constexpr int MINB = (QEG && DIM == 3) ? EDG_CORR_MINB_3D : (DIM == 2 ? EDG_CORR_MINB_2D : 1);
  static constexpr size_t BYTES = sizeof(double) * (2 * STAGE + TB + NV) +
                                  sizeof(unsigned long long) * (1 + CPB + CPB + 2) +
                                  sizeof(unsigned) * (((2 * DIM * CPB + 1) & ~1));
};

template <int KIND, int DIM, int N, bool GRID = true>
__global__ void __launch_bounds__(CorrPipe<KIND, DIM, N, GRID>::THREADS, CorrPipe<KIND, DIM, N, GRID>::MINB)
corrector_grid_pipe_kernel(const CorrArgs A) {
  const TraceScope trace_scope(A.trace);
  using P = Pde<KIND, DIM>;
  using C = CorrPipe<KIND, DIM, N, GRID>;
  constexpr int M = C::M, NPC = C::NPC, NF = C::NF, CPB = C::CPB, THREADS = C::THREADS, TRC = C::TRC;
  constexpr int FPC = 2 * DIM * M * NF;     // neighbour doubles per cell (= TRC)
  constexpr int TOT = 2 * DIM * NF;         // face points per cell

  extern __shared__ __align__(16) double smem[];
  double* const sStage = smem;                          // [2][STAGE]
  double* const sJump = smem + 2 * C::STAGE;            // [CPB][2d][M][NF]
  double* const sV = sJump + C::TB;                     // [2d][N] lift vectors (grid) / [CPB][2d][N] (adaptive)
  unsigned long long* const sLam = reinterpret_cast<unsigned long long*>(sV + C::NV);   // [1] CTA lambda max
  unsigned long long* const sLamC = sLam + 1;           // [CPB] per-cell lambda (adaptive)
  unsigned long long* const sFlag = sLamC + CPB;        // [CPB] non-finite flags
  unsigned* const sNan = reinterpret_cast<unsigned*>(sFlag + CPB);   // [2][DIM][CPB] NaN-axis flags
  unsigned long long* const sBar = reinterpret_cast<unsigned long long*>(sNan + ((2 * DIM * CPB + 1) & ~1));   // [2] stage mbarriers

  const int tid = threadIdx.x;
  const int slot = tid / NPC;
  const int node = tid - slot * NPC;
  const int n = A.grid_n;
  const int ngroups = (A.ncells - A.cell_base + CPB - 1) / CPB;   // cells [cell_base, ncells)

  // lift vectors v[a][s][i] = (sign * l_i(s)) / (w_i * h_a)   (kernels.py:190-191)
  auto lift = [&](int i, const double* e) {
    const int fs = i / N, j = i % N;
    const int a = fs >> 1, s = fs & 1;
    const double tr = A.basis[(s ? EDG_BASIS_TR(N) : EDG_BASIS_TL(N)) + j];
    const double sg = s ? 1.0 : -1.0;
    return __ddiv_rn(__dmul_rn(sg, tr), __dmul_rn(A.basis[EDG_BASIS_W(N) + j], e[a]));
  };
  if constexpr (GRID)
    for (int i = tid; i < 2 * DIM * N; i += THREADS) sV[i] = lift(i, A.edges);
  if (tid == 0) *sLam = 0ull;
  for (int i = tid; i < CPB; i += THREADS) sLamC[i] = 0ull;
  for (int i = tid; i < CPB; i += THREADS) sFlag[i] = 0ull;
  for (int i = tid; i < 2 * DIM * CPB; i += THREADS) sNan[i] = 0u;

  // per-thread constants: node coordinates, face point of the node on each
  // axis, and the lane mask of this thread's cell segment
  int ix[DIM], fpt[DIM];
  {
    int t = node;
#pragma unroll
    for (int a = DIM - 1; a >= 0; --a) {
      ix[a] = t % N;
      t /= N;
    }
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
      const int st = ipow(N, DIM - 1 - a);
      fpt[a] = (node / (st * N)) * st + (node % st);
    }
  }
    FastDiv fdn, fdn2;
  fdn.init((unsigned)n);
  fdn2.init((unsigned)n * (unsigned)(DIM == 3 ? n : 1));

  // issue the copies of group g into stage buffer st; the neighbour face
  // blocks (M * NF contiguous doubles each) go one warp per block
  // The three contiguous blocks go through the bulk-copy (TMA) engine when
  // 16-byte aligned and sized (one instruction each, completion counted on
  // the stage's mbarrier); otherwise cooperative cp.async.
  // L2 priorities (EDG_CORR_L2HINT): q_end and trace_f are read once
  // (evict_first), the own trace_q block is read again by the 2d neighbours
  // -- the i0 neighbours a whole plane of cells later (evict_last), so that
  // re-read finds it in L2 instead of DRAM
#ifndef EDG_CORR_L2HINT
#define EDG_CORR_L2HINT 1
#endif
  const unsigned long long pol_first = l2_policy_evict_first(), pol_last = l2_policy_evict_last();
  auto bulk_copy = [&](int i, void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    if (EDG_CORR_L2HINT && GRID)
      bulk_g2s_hint(dst, src, bytes, bar, i == 1 ? pol_last : pol_first);
    else
      bulk_g2s(dst, src, bytes, bar);
  };
  auto load_group = [&](int g, double* st, unsigned long long* bar) {
    const int c0 = A.cell_base + g * CPB;
    const int nc = min(CPB, A.ncells - c0);
    constexpr int NBK = C::NB;   // contiguous blocks: q_end, (trace_q,) trace_f
    constexpr int B0 = C::QEG ? 1 : 0;   // q_end not staged
    const double* srcs[3] = {A.q_end + (size_t)c0 * M * NPC, GRID ? A.trace_q + (size_t)c0 * TRC : A.trace_f + (size_t)c0 * TRC,
                             A.trace_f + (size_t)c0 * TRC};
    double* dsts[3] = {st, st + C::QE, st + C::QE + C::TB};
    const int cnt[3] = {nc * M * NPC, nc * TRC, nc * TRC};
    unsigned bulk_bytes = 0;
    bool bulk[3] = {false, false, false};
#pragma unroll
    for (int i = B0; i < NBK; ++i) {
      bulk[i] = ((reinterpret_cast<uintptr_t>(srcs[i]) & 15) == 0) && ((cnt[i] * 8) % 16 == 0);
      if (bulk[i]) bulk_bytes += (unsigned)cnt[i] * 8u;
    }
    constexpr int BLK = M * NF;
    // uniform grids whose face blocks are 16-byte multiples (2-D p = 5 / p = 3):
    // every copy of the group -- the contiguous blocks and the 2d neighbour
    // face blocks -- goes through the bulk-copy engine.  The expected bytes
    // are registered (no arrival) before any copy is issued, copies are issued
    // by one thread per block, and thread 0 arrives afterwards.
    if constexpr (GRID && (BLK * 8) % 16 == 0 && (TRC * 8) % 16 == 0) {
      bool all = (reinterpret_cast<uintptr_t>(A.trace_q) & 15) == 0;
#pragma unroll
      for (int i = B0; i < NBK; ++i) all = all && bulk[i];
      if (all) {
        if (tid == 0) mbar_expect_tx(bar, bulk_bytes + (unsigned)(nc * 2 * DIM * BLK * 8));
        __syncthreads();
        if (tid == 0) {
#pragma unroll
          for (int i = B0; i < NBK; ++i) bulk_copy(i, dsts[i], srcs[i], (unsigned)cnt[i] * 8u, bar);
        }
        double* nq = st + C::QE + (C::NB - 1) * C::TB;
        for (int bi = tid; bi < nc * 2 * DIM; bi += THREADS) {
          const int sl = bi / (2 * DIM), fs = bi - sl * (2 * DIM);
          const int a = fs >> 1, s = fs & 1;
          const unsigned cell = (unsigned)(c0 + sl);
          const unsigned q = a == DIM - 1 ? cell : (a == DIM - 2 ? fdn.div(cell) : fdn2.div(cell));
          const int ia = (int)(q - fdn.div(q) * (unsigned)n);
          const int stride = a == DIM - 1 ? 1 : (a == DIM - 2 ? n : n * n);
          int j = ia + (s ? 1 : -1);
          if (j < 0 || j >= n) j = A.periodic ? (j < 0 ? n - 1 : 0) : -1;
          const double* src = j >= 0 ? A.trace_q + (size_t)((int)cell + (j - ia) * stride) * TRC + (size_t)(2 * a + (1 - s)) * BLK
                                     : A.trace_q + (size_t)cell * TRC + (size_t)fs * BLK;
          bulk_g2s(nq + (sl * 2 * DIM + fs) * BLK, src, (unsigned)(BLK * 8), bar);
        }
        if (tid == 0) mbar_arrive(bar);
        return;
      }
    }
    if (tid == 0) {
      mbar_arrive_expect_tx(bar, bulk_bytes);
#pragma unroll
      for (int i = B0; i < NBK; ++i)
        if (bulk[i]) bulk_copy(i, dsts[i], srcs[i], (unsigned)cnt[i] * 8u, bar);
    }
#pragma unroll
    for (int i = B0; i < NBK; ++i)
      if (!bulk[i]) cp_block<THREADS>(dsts[i], srcs[i], cnt[i], tid);
    double* nq = st + C::QE + (C::NB - 1) * C::TB;
    constexpr int NW = THREADS / 32;
    const int warp = tid >> 5, lane = tid & 31;
    for (int bi = warp; bi < nc * 2 * DIM; bi += NW) {
      const int sl = bi / (2 * DIM), fs = bi - sl * (2 * DIM);
      double* dst = nq + (sl * 2 * DIM + fs) * BLK;
      if constexpr (!GRID) {
        // adaptive: the face outcome owning this side (missing: NaN in phase 1)
        const int fidx = __ldg(A.side_face + (size_t)(c0 + sl) * 2 * DIM + fs);
        if (fidx >= 0) {
          const double* src = A.outcomes + (size_t)fidx * BLK;
          if (((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {
            for (int i = lane; i < BLK / 2; i += 32) cp_async16(dst + 2 * i, src + 2 * i);
            if ((BLK & 1) && lane == 0) cp_async8(dst + BLK - 1, src + BLK - 1);
          } else {
            for (int i = lane; i < BLK; i += 32) cp_async8(dst + i, src + i);
          }
        }
        continue;
      }
      const int a = fs >> 1, s = fs & 1;
      const unsigned cell = (unsigned)(c0 + sl);
      const unsigned q = a == DIM - 1 ? cell : (a == DIM - 2 ? fdn.div(cell) : fdn2.div(cell));
      const int ia = (int)(q - fdn.div(q) * (unsigned)n);
      const int stride = a == DIM - 1 ? 1 : (a == DIM - 2 ? n : n * n);
      int j = ia + (s ? 1 : -1);
      if (j < 0 || j >= n) j = A.periodic ? (j < 0 ? n - 1 : 0) : -1;
      // neighbour's opposite face, or (outflow) the cell's own trace
      const double* src = j >= 0 ? A.trace_q + (size_t)((int)cell + (j - ia) * stride) * TRC + (size_t)(2 * a + (1 - s)) * BLK
                                 : A.trace_q + (size_t)cell * TRC + (size_t)fs * BLK;
      if (((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {
        for (int i = lane; i < BLK / 2; i += 32) cp_async16(dst + 2 * i, src + 2 * i);
        if ((BLK & 1) && lane == 0) cp_async8(dst + BLK - 1, src + BLK - 1);
      } else {
        for (int i = lane; i < BLK; i += 32) cp_async8(dst + i, src + i);
      }
    }
  };

  double lam_run = 0.0;                 // running max of lam_cell over this thread's cells (grid)
  unsigned long long best = DT_EMPTY;   // running minimum candidate (adaptive, threads < CPB)
  const unsigned segmask = lane_range_mask(slot * NPC, (slot + 1) * NPC);
  unsigned int nonfinite = 0u;

  if (tid == 0) {
    mbar_init(sBar, 1);
    mbar_init(sBar + 1, 1);
    mbar_fence_init();
  }
  __syncthreads();
  int g = blockIdx.x;
  if (g < ngroups) load_group(g, sStage, sBar);
  cp_async_commit();
  for (int it = 0; g < ngroups; g += gridDim.x, ++it) {
    double* const cur = sStage + (it & 1) * C::STAGE;
    const int gn = g + gridDim.x;
    if (gn < ngroups) load_group(gn, sStage + ((it + 1) & 1) * C::STAGE, sBar + ((it + 1) & 1));
    cp_async_commit();
    cp_async_wait1();                          // own cp.async copies of this group
    mbar_wait(sBar + (it & 1), (it >> 1) & 1);  // bulk copies of this group
    __syncthreads();

    const int cell = A.cell_base + g * CPB + slot;
    const bool has_cell = slot < CPB && cell < A.ncells;
    const bool cell_ok = A.cell_base + g * CPB < A.ncells;   // (WIDE: one cell, every thread in phase 1)
    const double* qe = cur;
    // QEG: this node's q_end straight from global memory, issued before the
    // face phase so the loads overlap it
    double qeg[M];
    if constexpr (C::QEG) {
#pragma unroll
      for (int k = 0; k < M; ++k)
        qeg[k] = has_cell ? (EDG_CORR_L2HINT ? __ldcs(A.q_end + (size_t)cell * M * NPC + (size_t)k * NPC + node)
                                             : __ldg(A.q_end + (size_t)cell * M * NPC + (size_t)k * NPC + node))
                          : 0.0;
    }
    const double* tq = cur + C::QE;
    const double* tf = cur + C::QE + (GRID ? C::TB : 0);
    const double* nq = cur + C::QE + (C::NB - 1) * C::TB;
    if constexpr (!GRID) {
      // per-cell lift vectors of this group (cell edges may differ)
      for (int i = tid; i < CPB * 2 * DIM * N; i += THREADS) {
        const int sl = i / (2 * DIM * N);
        const int c = A.cell_base + g * CPB + sl;
        if (c < A.ncells) sV[i] = lift(i - sl * 2 * DIM * N, A.edges + (A.edges_per_cell ? (size_t)c * DIM : 0));
      }
    }
    if (!GRID && has_cell) {
      // phase 1 (adaptive): outcome - trace_f, outcome gathered by side_face
      for (int f2 = node; f2 < TOT; f2 += NPC) {
        const int fs = f2 / NF, f = f2 - fs * NF;
        const int b = slot * TRC + fs * M * NF + f;
        const bool have = __ldg(A.side_face + (size_t)cell * 2 * DIM + fs) >= 0;
        if (!have) atomicOr(A.status, 2u);
#pragma unroll
        for (int k = 0; k < M; ++k)
          sJump[b + k * NF] =
              __dsub_rn(have ? nq[b + k * NF] : __longlong_as_double(0x7FF8000000000000ll), tf[b + k * NF]);
      }
    }
    // phase 1: Rusanov outcome - trace_f on the 2d faces (corrector_kernel order)
    if (GRID && (C::WIDE ? cell_ok : has_cell)) {
      for (int f2 = C::WIDE ? tid : node; f2 < TOT; f2 += C::WIDE ? THREADS : NPC) {
        const int fs = f2 / NF, f = f2 - fs * NF;
        const int a = fs >> 1, s = fs & 1;
        // face oriented along +a: lo = lower cell's (a,1) trace, hi = upper
        // cell's (a,0).  A warp's face points span two sides, so the sides
        // are chosen by address (one Rusanov evaluation per warp, no
        // divergent second pass)
        double lo[M], hi[M], out[M];
        const int b = (C::WIDE ? 0 : slot) * TRC + fs * M * NF + f;
        const double* const plo = s == 1 ? tq : nq;
        const double* const phi = s == 1 ? nq : tq;
#pragma unroll
        for (int k = 0; k < M; ++k) {
          lo[k] = plo[b + k * NF];
          hi[k] = phi[b + k * NF];
        }
        rusanov<KIND, DIM>(lo, hi, a, 1, A.pp, out);
#pragma unroll
        for (int k = 0; k < M; ++k) sJump[b + k * NF] = __dsub_rn(out[k], tf[b + k * NF]);
      }
    }
    __syncthreads();
    // phase 2: Q = q_end - sum v (x) jump in the reference (a, s) order
    double qn[M];
    bool finite = true;
#pragma unroll
    for (int k = 0; k < M; ++k) qn[k] = C::QEG ? qeg[k] : (has_cell ? qe[(slot * M + k) * NPC + node] : 0.0);
    if (has_cell) {
#pragma unroll
      for (int a = 0; a < DIM; ++a) {
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          const double v = sV[(GRID ? 0 : slot * 2 * DIM * N) + (2 * a + s) * N + ix[a]];
#pragma unroll
          for (int k = 0; k < M; ++k)
            qn[k] = __dsub_rn(qn[k], __dmul_rn(v, sJump[slot * TRC + ((2 * a + s) * M + k) * NF + fpt[a]]));
        }
      }
      double* qo = A.q_out + (size_t)cell * M * NPC + node;
#pragma unroll
      for (int k = 0; k < M; ++k) {
        if (EDG_CORR_L2HINT && GRID)
          __stcs(qo + (size_t)k * NPC, qn[k]);
        else
          qo[(size_t)k * NPC] = qn[k];
        finite = finite && (fabs(qn[k]) <= 1.7976931348623157e308);
      }
    }
    // next-step dt: on a uniform grid every cell shares h, so the minimum of
    // the per-cell candidates h / ((2p+1) lam_cell) is the candidate of the
    // largest lam_cell (division and the positive scaling are monotone, the
    // bits are the same).  lam_cell = python max over the axes whose
    // NaN-propagating node max is not NaN (kernels.py:267-281); an axis is
    // NaN for the cell iff some node's lambda on it is NaN, which a per-cell,
    // per-axis shared flag records.  Each node then folds max over its cell's
    // non-NaN axes into a per-thread running max (no per-group reduction).
    double lnode[DIM];
    unsigned* const nanf = sNan + (it & 1) * DIM * CPB;
    if (A.dt_slots && has_cell) {
      const auto pr = P::parts(qn, A.pp);
      P::lam_all(qn, pr, A.pp, lnode);
#pragma unroll
      for (int a = 0; a < DIM; ++a)
        if (lnode[a] != lnode[a]) nanf[a * CPB + slot] = 1u;
    }
    if (has_cell && !finite) sFlag[slot] = 1ull;
    __syncthreads();
    double lam = 0.0;
    if (A.dt_slots && has_cell) {
#pragma unroll
      for (int a = 0; a < DIM; ++a)
        if (nanf[a * CPB + slot] == 0u) lam = python_max(lam, lnode[a]);
      lam_run = lam > lam_run ? lam : lam_run;
    }
    if (!GRID && A.dt_slots) {
      // per-cell h: per-cell candidates (one NaN-free segmented max per cell)
      seg_max_redux(sLamC, has_cell ? slot : -1, segmask, (unsigned long long)__double_as_longlong(lam));
      __syncthreads();
      if (tid < CPB) {
        const int c = A.cell_base + g * CPB + tid;
        const double lc = __longlong_as_double((long long)sLamC[tid]);
        if (c < A.ncells && lc > 0.0) {
          const unsigned long long cand = (unsigned long long)__double_as_longlong(
              dt_candidate(A.hmin[A.edges_per_cell ? c : 0], A.order, lc));
          best = cand < best ? cand : best;
        }
        sLamC[tid] = 0ull;
      }
    }
    if (tid < CPB) {
      const int c = A.cell_base + g * CPB + tid;
      if (c < A.ncells && sFlag[tid]) ++nonfinite;
      sFlag[tid] = 0ull;
      // the other parity's flags are next written after this group's barriers
#pragma unroll
      for (int a = 0; a < DIM; ++a) sNan[((it + 1) & 1) * DIM * CPB + a * CPB + tid] = 0u;
    }
  }
  cp_async_wait1();   // (only empty groups can be outstanding here)
  if (tid < CPB && A.status && nonfinite) atomicAdd(A.status + 1, nonfinite);
  if (!GRID) {
    if (tid < CPB && A.dt_slots && best != DT_EMPTY) atomicMin(A.dt_slots + (blockIdx.x * CPB + tid) % EDG_DT_SLOTS, best);
  } else if (A.dt_slots) {
    // CTA max of the running maxima (non-negative, NaN-free: bit order = value order)
    unsigned long long key = (unsigned long long)__double_as_longlong(lam_run);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long v = __shfl_xor_sync(0xffffffffu, key, o);
      key = v > key ? v : key;
    }
    if ((tid & 31) == 0 && key) atomicMax(sLam, key);
    __syncthreads();
    if (tid == 0) {
      const double lam = __longlong_as_double((long long)*sLam);
      if (lam > 0.0)
        atomicMin(A.dt_slots + blockIdx.x % EDG_DT_SLOTS,
                  (unsigned long long)__double_as_longlong(dt_candidate(A.hmin[0], A.order, lam)));
    }
  }
}

}  // namespace edg
