// Face Riemann + corrector kernels -- replace kernels.py:162-193 and the
// hanging-face transfer of transfer.py:59-96.
//
// Corrector (kernels.py:176-193), per cell c, node x, component k:
//     Q = q_end - sum_{a,s} v_{a,s}[x_a] * (outcome_{a,s}[x without a] - trace_f_{a,s}[...])
//     v_{a,s} = (sign_s * l(s)) / (w * h_a)
// evaluated in the reference's (a, s) order with non-contracted multiply /
// subtract, so it is bit-identical to numpy for identical inputs.  Phase 1
// (threads over the 2d * n^(d-1) face points of each cell) forms the jumps in
// shared memory -- computing the Rusanov outcome inline from the neighbour's
// trace in the fused Cartesian mode -- and phase 2 (one thread per node)
// applies them.  Phase 3 folds the next step's admissible-dt candidate
// (kernels.py:267-281) into the same pass over the new state.
#pragma once
#include "edg_common.cuh"

namespace edg {

struct CorrArgs {
  const double* basis;
  int32_t ncells;           // end of the cell range (exclusive)
  int32_t cell_base;        // first cell of the range (0: all cells)
  int32_t order;
  const double* q_end;
  const double* trace_q;
  const double* trace_f;
  const int32_t* nbr;
  int32_t grid_n;           // > 0: uniform row-major grid_n^DIM mesh, neighbours by arithmetic
  int32_t periodic;
  const int32_t* side_face;
  const double* outcomes;
  const double* edges;
  int32_t edges_per_cell;
  double* q_out;
  unsigned long long* dt_slots;
  const double* hmin;
  uint32_t* status;
  PdeParams pp;
  unsigned long long* trace;   // optional launch-trace slot (TraceScope)
};

template <int DIM, int N>
struct CorrCfg {
  static constexpr int NPC = ipow(N, DIM);
  static constexpr int NF = ipow(N, DIM - 1);
  static constexpr int TARGET = 256;
  static constexpr int CPB = NPC >= TARGET ? 1 : (TARGET / NPC);
  static constexpr int THREADS = ((CPB * NPC + 31) / 32) * 32 < 64 ? 64 : ((CPB * NPC + 31) / 32) * 32;
};

template <int KIND, int DIM, int N>
struct CorrSmem {
  using C = CorrCfg<DIM, N>;
  static constexpr int M = Pde<KIND, DIM>::M;
  static constexpr size_t BYTES = sizeof(double) * (C::CPB * 2 * DIM * M * C::NF + C::CPB * 2 * DIM * N) +
                                  sizeof(unsigned long long) * (C::CPB * DIM + C::CPB) + sizeof(unsigned) * DIM * C::CPB;
};

template <int KIND, int DIM, int N, bool FUSED>
__global__ void __launch_bounds__(CorrCfg<DIM, N>::THREADS) corrector_kernel(const CorrArgs A) {
  const TraceScope trace_scope(A.trace);
  using P = Pde<KIND, DIM>;
  using Cf = CorrCfg<DIM, N>;
  constexpr int M = P::M;
  constexpr int NPC = Cf::NPC, NF = Cf::NF, CPB = Cf::CPB;
  constexpr int TRC = 2 * DIM * M * NF;     // trace doubles per cell

  extern __shared__ __align__(16) double smem[];
  double* sJump = smem;                                   // [CPB][2d][M][NF]
  double* sV = sJump + CPB * TRC;                         // [CPB][2d][N]
  unsigned long long* sLam = reinterpret_cast<unsigned long long*>(sV + CPB * 2 * DIM * N);  // [CPB][DIM]
  unsigned long long* sBest = sLam + CPB * DIM;           // [CPB]

  const int tid = threadIdx.x;
  const int slot = tid / NPC;
  const int node = tid - slot * NPC;
  const int cell = A.cell_base + blockIdx.x * CPB + slot;   // cells [cell_base, ncells)
  const bool has_cell = slot < CPB && cell < A.ncells;

  if (tid < CPB * DIM) sLam[tid] = 0ull;
  if (tid < CPB) sBest[tid] = 0ull;   // doubles as the per-cell non-finite flag until phase 3
  if (tid < CPB * DIM) reinterpret_cast<unsigned*>(sBest + CPB)[tid] = 0u;   // NaN-axis flags
  // q_end of this node, prefetched so its loads overlap the face gathers
  double qn[M];
  const size_t cb = (size_t)cell * M * NPC;
#pragma unroll
  for (int k = 0; k < M; ++k) qn[k] = has_cell ? __ldg(A.q_end + cb + (size_t)k * NPC + node) : 0.0;
  // lift vectors v[a][s][i] = (sign * l_i(s)) / (w_i * h_a)   (kernels.py:190-191)
  if (has_cell) {
    const double* e = A.edges + (A.edges_per_cell ? (size_t)cell * DIM : 0);
    for (int i = node; i < 2 * DIM * N; i += NPC) {
      const int fs = i / N, j = i % N;
      const int a = fs >> 1, s = fs & 1;
      const double tr = A.basis[(s ? EDG_BASIS_TR(N) : EDG_BASIS_TL(N)) + j];
      const double sg = s ? 1.0 : -1.0;
      sV[slot * 2 * DIM * N + i] = __ddiv_rn(__dmul_rn(sg, tr), __dmul_rn(A.basis[EDG_BASIS_W(N) + j], e[a]));
    }
    // phase 1: jumps outcome - trace_f on the 2d faces.  All global loads of
    // a thread's (at most IPT) face points are issued before any arithmetic.
    const size_t tb = (size_t)cell * TRC;
    constexpr int TOT = 2 * DIM * NF;
    constexpr int IPT = (TOT + NPC - 1) / NPC;
    // hoist all items of a thread when that costs few registers; otherwise one
    // item at a time (3-D p=4: hoisting two items lost occupancy, measured)
    constexpr int GRP = (3 * M * IPT <= 24) ? IPT : 1;
#pragma unroll 1
    for (int g0 = 0; g0 < IPT; g0 += GRP) {
    double mine[GRP][M], theirs[GRP][M], tfv[GRP][M];
#pragma unroll
    for (int i = 0; i < GRP; ++i) {
      const int it = node + (g0 + i) * NPC;
      if (it < TOT) {
        const int fs = it / NF, f = it - fs * NF;
        const int a = fs >> 1, s = fs & 1;
#pragma unroll
        for (int k = 0; k < M; ++k) tfv[i][k] = __ldg(A.trace_f + tb + ((size_t)fs * M + k) * NF + f);
        if (FUSED) {
          int nb;
          if (A.grid_n > 0) {
            // uniform row-major N^DIM grid: neighbour by index arithmetic
            const int n = A.grid_n;
            int stride = 1;
            for (int t = DIM - 1; t > a; --t) stride *= n;
            const int ia = (cell / stride) % n;
            int j = ia + (s ? 1 : -1);
            if (j < 0 || j >= n) j = A.periodic ? (j + n) % n : -1;
            nb = j < 0 ? -1 : cell + (j - ia) * stride;
          } else {
            nb = __ldg(A.nbr + (size_t)cell * 2 * DIM + fs);
          }
#pragma unroll
          for (int k = 0; k < M; ++k) mine[i][k] = __ldg(A.trace_q + tb + ((size_t)fs * M + k) * NF + f);
          const size_t ob = nb >= 0 ? (size_t)nb * TRC + ((size_t)(2 * a + (1 - s)) * M) * NF + f
                                    : tb + ((size_t)fs * M) * NF + f;   // outflow ghost = own trace
#pragma unroll
          for (int k = 0; k < M; ++k) theirs[i][k] = __ldg(A.trace_q + ob + (size_t)k * NF);
        } else {
          const int fidx = __ldg(A.side_face + (size_t)cell * 2 * DIM + fs);
          if (fidx < 0) {
            atomicOr(A.status, 2u);
#pragma unroll
            for (int k = 0; k < M; ++k) mine[i][k] = __longlong_as_double(0x7FF8000000000000ll);
          } else {
#pragma unroll
            for (int k = 0; k < M; ++k) mine[i][k] = __ldg(A.outcomes + ((size_t)fidx * M + k) * NF + f);
          }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < GRP; ++i) {
      const int it = node + (g0 + i) * NPC;
      if (it < TOT) {
        const int fs = it / NF, f = it - fs * NF;
        const int a = fs >> 1, s = fs & 1;
        double out[M];
        if (FUSED) {
          // face oriented along +a: lo = lower cell's (a,1) trace, hi = upper cell's (a,0)
          // (sides chosen by value: a warp's face points span two sides, one
          // Rusanov evaluation serves both instead of a divergent second pass)
          double lo[M], hi[M];
#pragma unroll
          for (int k = 0; k < M; ++k) {
            lo[k] = s == 1 ? mine[i][k] : theirs[i][k];
            hi[k] = s == 1 ? theirs[i][k] : mine[i][k];
          }
          rusanov<KIND, DIM>(lo, hi, a, 1, A.pp, out);
        } else {
#pragma unroll
          for (int k = 0; k < M; ++k) out[k] = mine[i][k];
        }
#pragma unroll
        for (int k = 0; k < M; ++k) sJump[slot * TRC + (fs * M + k) * NF + f] = __dsub_rn(out[k], tfv[i][k]);
      }
    }
    }
  }
  __syncthreads();
  // phase 2: Q = q_end - sum v (x) jump, reference (a, s) order
  bool finite = true;
  if (has_cell) {
    int ix[DIM];
    int t = node;
#pragma unroll
    for (int a = DIM - 1; a >= 0; --a) {
      ix[a] = t % N;
      t /= N;
    }
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
      const int st = ipow(N, DIM - 1 - a);
      const int f = (node / (st * N)) * st + (node % st);     // face point of this node
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const double v = sV[slot * 2 * DIM * N + (2 * a + s) * N + ix[a]];
#pragma unroll
        for (int k = 0; k < M; ++k)
          qn[k] = __dsub_rn(qn[k], __dmul_rn(v, sJump[slot * TRC + ((2 * a + s) * M + k) * NF + f]));
      }
    }
#pragma unroll
    for (int k = 0; k < M; ++k) {
      A.q_out[cb + (size_t)k * NPC + node] = qn[k];
      finite = finite && (fabs(qn[k]) <= 1.7976931348623157e308);
    }
  }
  // next-step dt candidate (kernels.py:267-281): lam_cell = python max over
  // the axes whose NaN-propagating node max is not NaN.  A per-(axis, cell)
  // shared flag records NaN axes; every node then contributes the max over
  // its cell's non-NaN axes, and one NaN-free maximum per cell remains.
  double lnode[DIM];
  unsigned* const sNan = reinterpret_cast<unsigned*>(sBest + CPB);   // [DIM][CPB]
  if (A.dt_slots && has_cell) {
    const auto pr = P::parts(qn, A.pp);
    P::lam_all(qn, pr, A.pp, lnode);
#pragma unroll
    for (int a = 0; a < DIM; ++a)
      if (lnode[a] != lnode[a]) sNan[a * CPB + slot] = 1u;
  }
  // per-cell non-finite flag (counted once per cell)
  if (has_cell && !finite) atomicOr(reinterpret_cast<unsigned int*>(sBest + slot), 1u);
  if (A.dt_slots || A.status) {
    __syncthreads();
    if (A.status && tid < CPB && (reinterpret_cast<unsigned int*>(sBest + tid)[0] & 1u))
      atomicAdd(A.status + 1, 1u);
  }
  if (A.dt_slots) {
    double lam = 0.0;
    if (has_cell) {
#pragma unroll
      for (int a = 0; a < DIM; ++a)
        if (sNan[a * CPB + slot] == 0u) lam = python_max(lam, lnode[a]);
    }
    const unsigned long long key = (unsigned long long)__double_as_longlong(lam);   // lam >= 0, no NaN
    if (A.edges_per_cell == 0) {
      // uniform h: min over cells of h/((2p+1) lam_cell) = candidate of the CTA max
      unsigned long long k2 = key;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long v = __shfl_xor_sync(0xffffffffu, k2, o);
        k2 = v > k2 ? v : k2;
      }
      if ((tid & 31) == 0 && k2) atomicMax(sLam, k2);
      __syncthreads();
      if (tid == 0) {
        const double lmax = __longlong_as_double((long long)*sLam);
        if (lmax > 0.0)
          atomicMin(A.dt_slots + (blockIdx.x % EDG_DT_SLOTS),
                    (unsigned long long)__double_as_longlong(dt_candidate(A.hmin[0], A.order, lmax)));
      }
    } else {
      const unsigned segmask = lane_range_mask(slot * NPC, (slot + 1) * NPC);
      seg_max_redux(sLam, has_cell ? slot : -1, segmask, key);
      __syncthreads();
      if (tid < CPB) {
        unsigned long long best = DT_EMPTY;
        const int c = A.cell_base + blockIdx.x * CPB + tid;
        if (c < A.ncells) {
          const double lc = __longlong_as_double((long long)sLam[tid]);
          if (lc > 0.0) best = (unsigned long long)__double_as_longlong(dt_candidate(A.hmin[c], A.order, lc));
        }
        sBest[tid] = best;
      }
      __syncthreads();
      if (tid == 0) {
        unsigned long long b = DT_EMPTY;
        for (int i = 0; i < CPB; ++i) b = sBest[i] < b ? sBest[i] : b;
        if (b != DT_EMPTY) atomicMin(A.dt_slots + (blockIdx.x % EDG_DT_SLOTS), b);
      }
    }
  }
}

// ------------------------------------------------------- hanging faces ----
struct FaceArgs {
  const double* basis;
  int32_t nfaces;
  const int32_t* axis;
  const int32_t* cell;      // [F][2]
  const int8_t* kind;       // [F][2]
  const int8_t* child_pos;  // [F][maxd][2]: transverse digits per chain level, coarsest first
  const int8_t* vdepth;     // [F] chain levels of the virtual side (null: 1)
  int32_t maxd;
  const double* trace_q;
  double* outcomes;
  PdeParams pp;
  unsigned long long* trace;   // optional launch-trace slot (TraceScope)
};

// trace of one side at face point f: own trace, or the coarse owner's trace
// evaluated at the leaf face's GL points (interpolate_to_virtual,
// transfer.py:59-79; axes contracted in order like _apply_axes,
// transfer.py:51-56).  Across a chain of `depth` levels the owner's trace is
// interpolated level by level (coarsest digit first), i.e. row f_t of
// I[d_depth] ... I[d_1] along each transverse axis t; at depth 1 the rows are
// those of I itself and the arithmetic is the one-level one.
template <int N>
__device__ __forceinline__ void chain_row(const double* interp, const int8_t* cp, int depth, int t, int ft,
                                          double (&R)[N]) {
  const double* I = interp + cp[2 * (depth - 1) + t] * N * N + ft * N;
#pragma unroll
  for (int l = 0; l < N; ++l) R[l] = I[l];
  for (int j = depth - 2; j >= 0; --j) {
    const double* J = interp + cp[2 * j + t] * N * N;
    double r2[N];
#pragma unroll
    for (int l = 0; l < N; ++l) {
      double v = 0.0;
#pragma unroll
      for (int m = 0; m < N; ++m) v = fma(R[m], J[m * N + l], v);
      r2[l] = v;
    }
#pragma unroll
    for (int l = 0; l < N; ++l) R[l] = r2[l];
  }
}

template <int DIM, int N, int M>
__device__ __forceinline__ void side_state(const double* tr, int kind, const int8_t* cp, int depth,
                                           const double* interp, int f, double* out) {
  constexpr int NF = ipow(N, DIM - 1);
  if (kind == 0) {
#pragma unroll
    for (int k = 0; k < M; ++k) out[k] = tr[k * NF + f];
    return;
  }
  if (DIM == 2) {
    double R[N];
    chain_row<N>(interp, cp, depth, 0, f, R);
#pragma unroll
    for (int k = 0; k < M; ++k) {
      double v = 0.0;
#pragma unroll
      for (int l = 0; l < N; ++l) v = fma(R[l], tr[k * NF + l], v);
      out[k] = v;
    }
  } else {
    const int f1 = f / N, f2 = f % N;
    double R1[N], R2[N];
    chain_row<N>(interp, cp, depth, 0, f1, R1);
    chain_row<N>(interp, cp, depth, 1, f2, R2);
#pragma unroll
    for (int k = 0; k < M; ++k) {
      double v = 0.0;
#pragma unroll
      for (int l2 = 0; l2 < N; ++l2) {
        double t = 0.0;
#pragma unroll
        for (int l1 = 0; l1 < N; ++l1) t = fma(R1[l1], tr[k * NF + l1 * N + l2], t);
        v = fma(R2[l2], t, v);
      }
      out[k] = v;
    }
  }
}

template <int KIND, int DIM, int N>
__global__ void __launch_bounds__(128) faces_rusanov_kernel(const FaceArgs A) {
  const TraceScope trace_scope(A.trace);
  using P = Pde<KIND, DIM>;
  constexpr int M = P::M;
  constexpr int NF = ipow(N, DIM - 1);
  __shared__ double sI[3 * N * N];
  for (int i = threadIdx.x; i < 3 * N * N; i += blockDim.x) sI[i] = A.basis[EDG_BASIS_INTERP(N) + i];
  __syncthreads();
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= (long long)A.nfaces * NF) return;
  const int fc = (int)(g / NF), f = (int)(g % NF);
  const int a = A.axis[fc];
  double st[2][M];
  int kinds[2];
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    kinds[s] = A.kind[2 * fc + s];
    if (kinds[s] != 2) {
      const int c = A.cell[2 * fc + s];
      // side s of the face is covered by the owner's face (a, 1 - s)
      const double* tr = A.trace_q + ((size_t)c * 2 * DIM + 2 * a + (1 - s)) * M * NF;
      side_state<DIM, N, M>(tr, kinds[s], A.child_pos + (size_t)fc * 2 * A.maxd, A.vdepth ? A.vdepth[fc] : 1, sI, f,
                            st[s]);
    }
  }
  if (kinds[0] == 2)
#pragma unroll
    for (int k = 0; k < M; ++k) st[0][k] = st[1][k];
  if (kinds[1] == 2)
#pragma unroll
    for (int k = 0; k < M; ++k) st[1][k] = st[0][k];
  double out[M];
  rusanov<KIND, DIM>(st[0], st[1], a, 1, A.pp, out);
#pragma unroll
  for (int k = 0; k < M; ++k) A.outcomes[((size_t)fc * M + k) * NF + f] = out[k];
}

// restrict_riemann accumulation (transfer.py:82-96): zero, then += each child
// restricted along the transverse axes, in child order.
template <int DIM, int N>
__global__ void __launch_bounds__(128) faces_restrict_kernel(const double* basis, int m, int nparents,
                                                             const int32_t* parent_face, const int32_t* children,
                                                             const int8_t* child_pos, double* outcomes,
                                                             unsigned long long* trace) {
  const TraceScope trace_scope(trace);
  constexpr int NF = ipow(N, DIM - 1);
  constexpr int NCH = ipow(3, DIM - 1);
  __shared__ double sR[3 * N * N];
  for (int i = threadIdx.x; i < 3 * N * N; i += blockDim.x) sR[i] = basis[EDG_BASIS_RESTR(N) + i];
  __syncthreads();
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= (long long)nparents * NF * m) return;
  const int p = (int)(g / (NF * m));
  const int rem = (int)(g % (NF * m));
  const int k = rem / NF, f = rem % NF;
  double acc = 0.0;
  for (int j = 0; j < NCH; ++j) {
    const int ch = children[p * NCH + j];
    const int8_t* cp = child_pos + 2 * ch;
    const double* src = outcomes + ((size_t)ch * m + k) * NF;
    double v = 0.0;
    if (DIM == 2) {
      const double* R = sR + cp[0] * N * N + f * N;
#pragma unroll
      for (int l = 0; l < N; ++l) v = fma(R[l], src[l], v);
    } else {
      const int f1 = f / N, f2 = f % N;
      const double* R1 = sR + cp[0] * N * N + f1 * N;
      const double* R2 = sR + cp[1] * N * N + f2 * N;
#pragma unroll
      for (int l2 = 0; l2 < N; ++l2) {
        double t = 0.0;
#pragma unroll
        for (int l1 = 0; l1 < N; ++l1) t = fma(R1[l1], src[l1 * N + l2], t);
        v = fma(R2[l2], t, v);
      }
    }
    acc = __dadd_rn(acc, v);
  }
  outcomes[((size_t)parent_face[p] * m + k) * NF + f] = acc;
}

// project_to_faces on a batch (kernels.py:73-79): out[c][2a+s][k][f] =
// sum_j l_j(s) vol[c][k][node(f, a, j)]
template <int DIM, int N>
__global__ void __launch_bounds__(128) project_faces_kernel(const double* basis, int m, int ncells,
                                                            const double* vol, double* out) {
  constexpr int NF = ipow(N, DIM - 1), NPC = ipow(N, DIM);
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= (long long)ncells * 2 * DIM * m * NF) return;
  const int c = (int)(g / (2 * DIM * m * NF));
  const int r = (int)(g % (2 * DIM * m * NF));
  const int fs = r / (m * NF), k = (r / NF) % m, f = r % NF;
  const int a = fs >> 1, s = fs & 1;
  const double* tv = basis + (s ? EDG_BASIS_TR(N) : EDG_BASIS_TL(N));
  const double* src = vol + ((size_t)c * m + k) * NPC;
  const int st = ipow(N, DIM - 1 - a);
  const int hi = f / st, lo = f - hi * st;
  double v = 0.0;
#pragma unroll
  for (int j = 0; j < N; ++j) v = fma(tv[j], src[hi * st * N + j * st + lo], v);
  out[g] = v;
}

// interpolate_face_trace / restrict_face_values on a batch (transfer.py:59-72)
template <int DIM, int N>
__global__ void __launch_bounds__(128) face_transfer_kernel(const double* basis, int m, int nfaces,
                                                            const double* in, const int8_t* child_pos,
                                                            int restrict_mode, double* out) {
  constexpr int NF = ipow(N, DIM - 1);
  __shared__ double sT[3 * N * N];
  const int off = restrict_mode ? EDG_BASIS_RESTR(N) : EDG_BASIS_INTERP(N);
  for (int i = threadIdx.x; i < 3 * N * N; i += blockDim.x) sT[i] = basis[off + i];
  __syncthreads();
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= (long long)nfaces * NF * m) return;
  const int fc = (int)(g / (NF * m));
  const int rem = (int)(g % (NF * m));
  const int k = rem / NF, f = rem % NF;
  const int8_t* cp = child_pos + 2 * fc;
  const double* src = in + ((size_t)fc * m + k) * NF;
  double v = 0.0;
  if (DIM == 2) {
    const double* T = sT + cp[0] * N * N + f * N;
#pragma unroll
    for (int l = 0; l < N; ++l) v = fma(T[l], src[l], v);
  } else {
    const int f1 = f / N, f2 = f % N;
    const double* T1 = sT + cp[0] * N * N + f1 * N;
    const double* T2 = sT + cp[1] * N * N + f2 * N;
#pragma unroll
    for (int l2 = 0; l2 < N; ++l2) {
      double t = 0.0;
#pragma unroll
      for (int l1 = 0; l1 < N; ++l1) t = fma(T1[l1], src[l1 * N + l2], t);
      v = fma(T2[l2], t, v);
    }
  }
  out[((size_t)fc * m + k) * NF + f] = v;
}

}  // namespace edg
