// hd_cell.cuh -- the fused cell kernel (element-centric loop, Alg. 1/Alg. 2) for sm_100a.
// Included by hd_kernels.cu (single translation unit with the __constant__ tables).
//
// Merged operator: M^-1 A = sum_i L_i along dim i, per line of dim i
//   (L_i u)_m = s * [ sum_q K[m][q] u_q + lam[m] (tau . u_nb) ],   s = a_i(z_line) dt / h_i,
// K = volume term + own-face upwind term (rows divided by w_m), lam/tau = the rank-1 lift of the UPWIND
// neighbour's trace (folded). The line speed s is applied to the line's values before the
// contraction: for a dim whose speed is constant on the mesh it is folded into the tables s K, s tau
// (kernel parameters: no extra instruction), otherwise the N values of each line are scaled once. A
// published trace is the scaled one, T = tau . (s u_nb), so the consumer's lift is lam[m] * T.
//
// One CTA iteration processes a GROUP of CT cells (static schedule, hd_sched.cpp); threads own, per
// phase, an n x n register tile of a cell over a pair of dims (P, Q) and contract both dims from
// registers. Two smem cell buffers alternate roles: the group's cells (U) and the phase accumulator
// (ACC); once every thread has read its last-phase tile, the next group's cells stream into the ACC
// buffer while the last phase computes, and the roles swap.
//
// Upwind traces come from the static schedule: the dim-0 carry of the previous step (smem), an in-group
// neighbour (smem), a trace published by an earlier unit (global, ready when its producer's progress
// flag -- read with ld.acquire -- says so), the halo buffer, or a direct read of the neighbour cell.
#pragma once
// Lean kernel: two CTAs per SM -- two cell buffers (U, accumulator; the next group's cells
// stream into U once every thread has read its last-phase tile), one dim-0 carry buffer, published / halo
// traces read from L2 in the phase instead of staged, <= 128 registers per thread. Used for d >= 4 with
// n <= 4 (the n = 5 tile does not fit 128 registers); HD_LEAN = 0 / 1 forces it off / on (experiments).
#ifndef HD_LEAN
#define HD_LEAN -1
#endif
#ifndef HD_LEAN_PF
#define HD_LEAN_PF 1
#endif
#ifndef HD_PF_PUB
#define HD_PF_PUB 1
#endif
#ifndef HD_PF_DIRECT
#define HD_PF_DIRECT 2
#endif
#ifndef HD_PF_DU
#define HD_PF_DU 2
#endif
#ifndef HD_FILL_EF
#define HD_FILL_EF 1
#endif
#ifndef HD_DYN
#define HD_DYN 1
#endif

namespace hd {

template <int D, int N>
__host__ __device__ constexpr bool lean() {
  return HD_LEAN == 1 || (HD_LEAN < 0 && D >= 4 && N <= 4);
}
constexpr bool kDyn = HD_DYN != 0;

// Shared-memory layout of a cell: element (d_0, ..., d_{D-1}) at sum_i d_i S_i -- ADDITIVE, so a thread's
// tile element is its rest offset plus a compile-time constant (base + immediate addressing). The padded
// strides (tools/smem_layout.py; pinned by tests/test_smem_layout.py) keep the layout injective (mixed
// radix), keep 16-byte pairs along dim 0 aligned (N even: S_i even for i >= 1) and make the tile accesses
// of every phase (nearly) bank-conflict free; other (D, N) keep the plain strides N^i.
struct CellStrides {
  int s[kMaxD];
};
template <int D, int N>
__host__ __device__ constexpr CellStrides cell_strides() {
  if constexpr (D == 3 && N == 4) return {{1, 4, 18}};
  else if constexpr (D == 3 && N == 5) return {{1, 5, 28}};
  else if constexpr (D == 4 && N == 4) return {{1, 4, 18, 76}};
  else if constexpr (D == 4 && N == 5) return {{1, 5, 25, 136}};
  else if constexpr (D == 5 && N == 2) return {{1, 2, 4, 8, 18}};
  else if constexpr (D == 5 && N == 3) return {{1, 3, 9, 27, 88}};
  else if constexpr (D == 5 && N == 4) return {{1, 4, 18, 76, 298}};
  else if constexpr (D == 5 && N == 5) return {{1, 5, 25, 133, 665}};
  else if constexpr (D == 6 && N == 2) return {{1, 2, 4, 8, 18, 36}};
  else if constexpr (D == 6 && N == 3) return {{1, 3, 9, 27, 81, 245}};
  else if constexpr (D == 6 && N == 4) return {{1, 4, 18, 76, 298, 1192}};
  else {
    CellStrides r{};
    int m = 1;
    for (int i = 0; i < D; ++i) {
      r.s[i] = m;
      m *= N;
    }
    return r;
  }
}
// doubles per cell in shared memory (even when N is even: 16-byte aligned cells)
template <int D, int N>
__host__ __device__ constexpr int cell_span() {
  constexpr CellStrides S = cell_strides<D, N>();
  int m = 0;
  for (int i = 0; i < D; ++i) m += (N - 1) * S.s[i];
  m += 1;
  return (N % 2 == 0 && m % 2) ? m + 1 : m;
}

template <int D, int N>
struct CGeo {
  static constexpr int ND = ipow(N, D);
  static constexpr int NDP = cell_span<D, N>();  // smem doubles per cell (padded layout)
  static constexpr int FN = ipow(N, D - 1);   // face points per face
  static constexpr int NT = ipow(N, D - 2);   // threads per cell
  static constexpr int NPH = (D + 1) / 2;     // phases
  // phase ph works on the dim pair (P, Q): (0, D-1), (1, 2), (3, 4); QA false: Q already done
  static constexpr __host__ __device__ int P(int ph) { return ph == 0 ? 0 : 2 * ph - 1; }
  static constexpr __host__ __device__ bool QA(int ph) { return ph == 0 || 2 * ph != D - 1; }
  static constexpr __host__ __device__ int Q(int ph) { return ph == 0 ? D - 1 : 2 * ph; }
  // one cell (two buffers) must fit the smem of one CTA: n^d <= 4096
  static constexpr bool OK = NT <= 256 && (2 * NDP + FN + NPH * 1024) * 8 + 1024 <= 227 * 1024;
};

// smem position of cell-local element x (runtime digits)
template <int D, int N>
__host__ __device__ __forceinline__ constexpr int swz(int x) {
  constexpr CellStrides S = cell_strides<D, N>();
  unsigned ux = (unsigned)x, p = 0;  // unsigned: digit extraction is a mask and a shift for N = 2^m
#pragma unroll
  for (int i = 0; i < D; ++i) {
    p += (ux % N) * (unsigned)S.s[i];
    ux /= N;
  }
  return (int)p;
}
// element T (compile-time offset whose digits are disjoint from the thread's rest offset R, sR = swz(R)):
// the layout is additive, so this folds to sR + constant
template <int D, int N>
__device__ __forceinline__ constexpr int sidx(int sR, int T) {
  return sR + swz<D, N>(T);
}

// HD_DEBUG builds: device-side checks that record into the mesh's error word (the host
// reports HD_ERR_STATE); release builds compile them out.
#ifdef HD_DEBUG
#define HD_DCHECK(p, cond, bit)                  \
  do {                                           \
    if (!(cond)) atomicOr((p).err, (bit));       \
  } while (0)
#else
#define HD_DCHECK(p, cond, bit) \
  do {                          \
  } while (0)
#endif

// HD_PROFILE builds (experiments only): lane 0 of every warp of CTAs 0 and 74 accumulates,
// per barrier site of the group loop, the cycles it waited at the barrier (clock64 at arrival; after the
// barrier a dependent smem read forces the deferred block) and the cycles between barriers; printed per
// warp at the end of the launch.
#ifdef HD_PROFILE
#define HD_PROF_DECL                                                                  \
  unsigned long long pf_t = clock64(), pf_wait[4] = {0, 0, 0, 0}, pf_work[4] = {0, 0, 0, 0}, pf_groups = 0; \
  unsigned long long pf_sub[3][6] = {}, pf_main[8] = {}, pf_m = 0;
#define HD_PF(ph) pf_sub[ph]
#define HD_MARK(k)                          \
  do {                                      \
    const unsigned long long t_ = clock64(); \
    pf_main[(k)] += t_ - pf_m;              \
    pf_m = t_;                              \
  } while (0)
#define HD_PROF_BAR(site)                                                              \
  do {                                                                                 \
    const unsigned long long ta_ = clock64();                                          \
    pf_work[site] += ta_ - pf_t;                                                       \
    __syncthreads();                                                                   \
    const unsigned long long tb_ = clock64() + *(volatile int *)smem_raw * 0;          \
    pf_wait[site] += tb_ - ta_;                                                        \
    pf_t = tb_;                                                                        \
    pf_m = tb_;                                                                        \
  } while (0)
#define HD_PROF_GROUP() ++pf_groups
#define HD_SUB_DECL unsigned long long sb_t = clock64();
#define HD_SUB(k)                                   \
  do {                                              \
    const unsigned long long t_ = clock64();        \
    if (pf_sub) pf_sub[(k)] += t_ - sb_t;           \
    sb_t = t_;                                      \
  } while (0)
#define HD_PROF_DUMP()                                                                                         \
  if ((blockIdx.x == 0 || blockIdx.x == 74) && (threadIdx.x & 31) == 0 && pf_groups)                           \
    printf("HDPROF cta %d warp %d | wait top %llu b0 %llu b1 %llu bL %llu | work ->top %llu ->b0 %llu ->b1 %llu " \
           "->bL %llu\n",                                                                                       \
           blockIdx.x, threadIdx.x >> 5, pf_wait[0] / pf_groups, pf_wait[1] / pf_groups, pf_wait[2] / pf_groups, \
           pf_wait[3] / pf_groups, pf_work[0] / pf_groups, pf_work[1] / pf_groups, pf_work[2] / pf_groups,       \
           pf_work[3] / pf_groups);                                                                              \
  if ((blockIdx.x == 0) && (threadIdx.x & 31) == 0 && pf_groups)                                              \
    for (int ph_ = 0; ph_ < 3; ++ph_)                                                                          \
      printf("HDSUB warp %d phase %d | loads %llu passP %llu passQ %llu trP+liftP %llu trQ+liftQ %llu store %llu\n", \
             threadIdx.x >> 5, ph_, pf_sub[ph_][0] / pf_groups, pf_sub[ph_][1] / pf_groups,                     \
             pf_sub[ph_][2] / pf_groups, pf_sub[ph_][3] / pf_groups, pf_sub[ph_][4] / pf_groups,                \
             pf_sub[ph_][5] / pf_groups);                                                               \
  if ((blockIdx.x == 0) && (threadIdx.x & 31) == 0 && pf_groups)                                              \
    printf("HDMAIN warp %d | stage %llu fetch %llu cells %llu ph0 %llu | flags %llu ph1 %llu | ph2 %llu resolve %llu\n", \
           threadIdx.x >> 5, pf_main[0] / pf_groups, pf_main[1] / pf_groups, pf_main[2] / pf_groups,               \
           pf_main[3] / pf_groups, pf_main[4] / pf_groups, pf_main[5] / pf_groups, pf_main[6] / pf_groups,        \
           pf_main[7] / pf_groups)
#else
#define HD_MARK(k) \
  do {             \
  } while (0)
#define HD_PROF_DECL
#define HD_PF(ph) nullptr
#define HD_PROF_BAR(site) __syncthreads()
#define HD_PROF_GROUP() \
  do {                  \
  } while (0)
#define HD_SUB_DECL
#define HD_SUB(k) \
  do {            \
  } while (0)
#define HD_PROF_DUMP() \
  do {                 \
  } while (0)
#endif

// Resolved schedule of one cell of a group (smem, double buffered; written by the lanes that own the
// group's (cell, dim) items, read by every thread of the cell).
struct CellInfo {
  double base[kMaxD];         // a_i at the cell's lower corner
  const double *tsrc[kMaxD];  // kSrcPub / kSrcHalo: the trace; kSrcDirect: the neighbour cell
  int cell;                   // local cell index
  int oslot;                  // published-trace slot of the cell
  unsigned char nb[kMaxD];    // kSrcGroup: neighbour slot
  unsigned char src[kMaxD], out[kMaxD], sg[kMaxD];
};

// per-thread, per-phase constants
struct ThreadPhase {
  double wP, wQ;  // sum over rest dims j of a_lin[P|Q][j] h_j xi_{m_j}
  double wr;      // |J| prod_{rest j} w_{m_j} (weak-form mass, A mode)
  int R;          // cell-local offset of the rest coordinates
};

__device__ __forceinline__ int ld_acquire(const int *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int *p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
// Drop a 128-byte L2 line without writing it back (its data becomes undefined).
__device__ __forceinline__ void discard_l2(const void *p) {
  asm volatile("discard.global.L2 [%0], 128;\n" ::"l"(p) : "memory");
}
// Bring a whole cell (contiguous, 16-byte multiple) into L2 ahead of its read.
__device__ __forceinline__ void prefetch_l2(const void *p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(bytes) : "memory");
}

// Line speed of the cell's lines along dim i (a_i depends only on the other coordinates):
// a_i(z) * dtfac / h_i = s0 + sl * xi_l, l = the line's node along the partner dim of the tile.
struct LineSpeed {
  double s0, sl;
};

// 1D tables of dim X, sign S: variable-speed dims use the unit-speed c_tab tables on scaled lines,
// constant-speed dims the prescaled kernel-parameter tables s K, s tau (compile-time offsets: the DFMA
// reads them as constant-bank operands).
template <int N, int X, int S, bool VAR>
__device__ __forceinline__ double kval(const CellParams &p, int a, int j) {
  if constexpr (VAR) return c_tab[N].K[S][a][j];
  else return p.Ks[((X * 2 + S) * N + a) * N + j];
}
template <int N, int X, int S, bool VAR>
__device__ __forceinline__ double tval(const CellParams &p, int j) {
  if constexpr (VAR) return c_tab[N].tau[S][j];
  else return p.Ts[(X * 2 + S) * N + j];
}

// The (scaled) trace of one line of dim X with values v and line speed s: T = sum_j tau_j (s v_j). Every
// trace source (producer pass, in-group smem, direct read, halo pack) evaluates exactly this sequence, so
// the source of a trace never changes its bits.
template <int N, int X, int S, bool VAR>
__device__ __forceinline__ double line_trace(const CellParams &p, const double (&v)[N], double s) {
  double us[N];
#pragma unroll
  for (int j = 0; j < N; ++j) us[j] = VAR ? s * v[j] : v[j];
  double t = tval<N, X, S, VAR>(p, 0) * us[0];
#pragma unroll
  for (int j = 1; j < N; ++j) t = fma(tval<N, X, S, VAR>(p, j), us[j], t);
  return t;
}

// Pass over the tile lines of dim P (tile index a; one line per partner digit b): the line's downwind
// trace t[b] and the volume + own-face contribution acc[a][b] (+)= sum_j (sK)[a][j] u[j][b].
template <int N, int X, int S, bool VAR, bool INIT>
__device__ __forceinline__ void pass_P(const CellParams &p, double (&acc)[N][N], const double (&uv)[N][N], LineSpeed ls,
                                       double (&t)[N]) {
#pragma unroll
  for (int b = 0; b < N; ++b) {
    const double sb = VAR ? fma(ls.sl, c_tab[N].xi[b], ls.s0) : 0.0;
    double us[N];
#pragma unroll
    for (int j = 0; j < N; ++j) us[j] = VAR ? sb * uv[j][b] : uv[j][b];
    double tr = tval<N, X, S, VAR>(p, 0) * us[0];
#pragma unroll
    for (int j = 1; j < N; ++j) tr = fma(tval<N, X, S, VAR>(p, j), us[j], tr);
    t[b] = tr;
#pragma unroll
    for (int j = 0; j < N; ++j)
#pragma unroll
      for (int a = 0; a < N; ++a) {
        if (INIT && j == 0) acc[a][b] = kval<N, X, S, VAR>(p, a, 0) * us[0];
        else acc[a][b] = fma(kval<N, X, S, VAR>(p, a, j), us[j], acc[a][b]);
      }
  }
}
// Same for dim Q (tile index b; one line per a).
template <int N, int X, int S, bool VAR>
__device__ __forceinline__ void pass_Q(const CellParams &p, double (&acc)[N][N], const double (&uv)[N][N], LineSpeed ls,
                                       double (&t)[N]) {
#pragma unroll
  for (int a = 0; a < N; ++a) {
    const double sa = VAR ? fma(ls.sl, c_tab[N].xi[a], ls.s0) : 0.0;
    double us[N];
#pragma unroll
    for (int j = 0; j < N; ++j) us[j] = VAR ? sa * uv[a][j] : uv[a][j];
    double tr = tval<N, X, S, VAR>(p, 0) * us[0];
#pragma unroll
    for (int j = 1; j < N; ++j) tr = fma(tval<N, X, S, VAR>(p, j), us[j], tr);
    t[a] = tr;
#pragma unroll
    for (int j = 0; j < N; ++j)
#pragma unroll
      for (int b = 0; b < N; ++b) acc[a][b] = fma(kval<N, X, S, VAR>(p, b, j), us[j], acc[a][b]);
  }
}
// run-time dispatch over (sign, variable speed): uniform per cell / per launch
template <int N, int X, bool INIT>
__device__ __forceinline__ void pass_P_any(const CellParams &p, double (&acc)[N][N], const double (&uv)[N][N], LineSpeed ls,
                                           double (&t)[N], int sg, int var) {
  if (var) {
    if (sg) pass_P<N, X, 1, true, INIT>(p, acc, uv, ls, t);
    else pass_P<N, X, 0, true, INIT>(p, acc, uv, ls, t);
  } else {
    if (sg) pass_P<N, X, 1, false, INIT>(p, acc, uv, ls, t);
    else pass_P<N, X, 0, false, INIT>(p, acc, uv, ls, t);
  }
}
template <int N, int X>
__device__ __forceinline__ void pass_Q_any(const CellParams &p, double (&acc)[N][N], const double (&uv)[N][N], LineSpeed ls,
                                           double (&t)[N], int sg, int var) {
  if (var) {
    if (sg) pass_Q<N, X, 1, true>(p, acc, uv, ls, t);
    else pass_Q<N, X, 0, true>(p, acc, uv, ls, t);
  } else {
    if (sg) pass_Q<N, X, 1, false>(p, acc, uv, ls, t);
    else pass_Q<N, X, 0, false>(p, acc, uv, ls, t);
  }
}

// Upwind trace of dim X for this thread's N face points from cell values: the line of face point l is
// v_j = src[j*SX + l*SY] (smem: additive layout via sidx; global: plain n^i strides), speed s0 + sl xi_l.
template <int D, int N, int X, int SX, int SY, int S, bool VAR, bool SMEM>
__device__ __forceinline__ void trace_cell_s(const CellParams &p, const double *src, int off, LineSpeed ls, double (&t)[N]) {
#pragma unroll
  for (int l = 0; l < N; ++l) {
    double v[N];
#pragma unroll
    for (int j = 0; j < N; ++j) {
      if constexpr (SMEM) v[j] = src[sidx<D, N>(off, j * SX + l * SY)];
      else v[j] = __ldg(src + off + j * SX + l * SY);
    }
    t[l] = line_trace<N, X, S, VAR>(p, v, VAR ? fma(ls.sl, c_tab[N].xi[l], ls.s0) : 0.0);
  }
}
template <int D, int N, int X, int SX, int SY, bool SMEM>
__device__ __forceinline__ void trace_cell(const CellParams &p, const double *src, int off, LineSpeed ls, int sg, int var,
                                           double (&t)[N]) {
  if (var) {
    if (sg) trace_cell_s<D, N, X, SX, SY, 1, true, SMEM>(p, src, off, ls, t);
    else trace_cell_s<D, N, X, SX, SY, 0, true, SMEM>(p, src, off, ls, t);
  } else {
    if (sg) trace_cell_s<D, N, X, SX, SY, 1, false, SMEM>(p, src, off, ls, t);
    else trace_cell_s<D, N, X, SX, SY, 0, false, SMEM>(p, src, off, ls, t);
  }
}

template <int N>
__device__ __forceinline__ void store_vec(double *dst, const double (&t)[N], bool global) {
  if constexpr (N % 2 == 0) {
#pragma unroll
    for (int j = 0; j < N; j += 2) {
      if (global) __stcg(reinterpret_cast<double2 *>(dst + j), make_double2(t[j], t[j + 1]));
      else *reinterpret_cast<double2 *>(dst + j) = make_double2(t[j], t[j + 1]);
    }
  } else {
#pragma unroll
    for (int j = 0; j < N; ++j) {
      if (global) __stcg(dst + j, t[j]);
      else dst[j] = t[j];
    }
  }
}
// N (even) values with the L2 evict_last policy: data this CTA reads back soon, to survive the streams
template <int N>
__device__ __forceinline__ void store_vec_keep(double *dst, const double (&t)[N]) {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol));
#pragma unroll
  for (int j = 0; j < N; j += 2)
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;\n" ::"l"(dst + j), "d"(t[j]), "d"(t[j + 1]), "l"(pol)
                 : "memory");
}
template <int N>
__device__ __forceinline__ void load_vec(const double *src, double (&t)[N], bool global) {
  if constexpr (N % 2 == 0) {
#pragma unroll
    for (int j = 0; j < N; j += 2) {
      const double2 v = global ? __ldcg(reinterpret_cast<const double2 *>(src + j))
                               : *reinterpret_cast<const double2 *>(src + j);
      t[j] = v.x;
      t[j + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int j = 0; j < N; ++j) t[j] = global ? __ldcg(src + j) : src[j];
  }
}

// Cell-local offset (dim-X digit 0) of face point f = N r + l of dim X in the phase layout of X: rest
// digits r (dims other than the phase pair, ascending), partner tile digit l.
template <int D, int N>
__device__ __forceinline__ int face_offset(int X, int f) {
  using G = CGeo<D, N>;
  const int ph = (X == 0 || X == D - 1) ? 0 : (X + 1) / 2;
  const int P = G::P(ph), Q = G::Q(ph);
  const int partner = X == P ? Q : P;
  int r = f / N;
  const int l = f - r * N;
  int R = 0, nj = 1;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    if (j != P && j != Q) {
      R += (r % N) * nj;
      r /= N;
    }
    nj *= N;
  }
  int sp = 1;
  for (int j = 0; j < partner; ++j) sp *= N;
  return R + l * sp;
}

// Per-thread phase constants for rest index r (speed offsets of the rest coordinates, weak-form mass).
template <int D, int N, int PH, bool MASS>
__device__ __forceinline__ void thread_phase(const CellParams &p, int r, ThreadPhase &tp) {
  using G = CGeo<D, N>;
  constexpr int P = G::P(PH), Q = G::Q(PH);
  int rr = r, R = 0, nj = 1;
  double wP = 0.0, wQ = 0.0, wr = p.jdet;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    if (j != P && j != Q) {
      const int m = rr % N;
      rr /= N;
      R += m * nj;
      wP = fma(p.a_lin[P][j] * p.h[j], c_tab[N].xi[m], wP);
      wQ = fma(p.a_lin[Q][j] * p.h[j], c_tab[N].xi[m], wQ);
      if constexpr (MASS) wr *= c_tab[N].w[m];
    }
    nj *= N;
  }
  tp.wP = wP;
  tp.wQ = wQ;
  tp.wr = wr;
  tp.R = R;
}
// speeds of the lines of dim X (phase partner Y) of a cell with corner speed `base`, for a thread with
// rest offset w: s = (base + w) * fac_X + slin[X][Y] xi_l (fac_X = dtfac / h_X, slin = a_lin[X][Y] h_Y fac_X,
// per-launch kernel parameters). The halo pack kernel evaluates the same expressions.
__device__ __forceinline__ LineSpeed line_speed(const CellParams &p, int X, int Y, double base, double w) {
  return LineSpeed{(base + w) * p.fac[X], p.slin[X][Y]};
}

// The per-thread constants of every phase, once per launch into this thread's column of the smem table
// read by run_phase: [PH][wP | wQ | wr | (R, sR)][256].
template <int D, int N, int MODE, int PH>
__device__ __forceinline__ void phase_entry(const CellParams &p, int r, double *ptab) {
  using G = CGeo<D, N>;
  ThreadPhase tp;
  thread_phase<D, N, PH, PH == G::NPH - 1 && (MODE == kModeAdvection || MODE == kModeAdvAcc)>(p, r, tp);
  double *pt = ptab + PH * 1024;
  const int tid = (int)threadIdx.x;
  pt[tid] = tp.wP;
  pt[256 + tid] = tp.wQ;
  pt[512 + tid] = tp.wr;
  reinterpret_cast<int2 *>(pt + 768)[tid] = make_int2(tp.R, swz<D, N>(tp.R));
}
template <int D, int N, int MODE>
__device__ __forceinline__ void phase_table(const CellParams &p, int r, double *ptab) {
  using G = CGeo<D, N>;
  phase_entry<D, N, MODE, 0>(p, r, ptab);
  if constexpr (G::NPH > 1) phase_entry<D, N, MODE, (G::NPH > 1 ? 1 : 0)>(p, r, ptab);
  if constexpr (G::NPH > 2) phase_entry<D, N, MODE, (G::NPH > 2 ? 2 : 0)>(p, r, ptab);
}

// Smem pointers of the thread's cell in the current group.
struct GroupBufs {
  const double *Ugrp;     // the group's cells (U buffer, slot 0)
  const double *U;        // this thread's cell
  double *A;              // this thread's cell's accumulator (the other buffer)
  const double *carry;    // this cell's incoming dim-0 carry (the previous step's downwind trace)
  double *carry_out;      // ... and the one this step produces (the other half of the double buffer)
};

// Upwind trace of dim X (tile stride SX, partner stride SY) from the source the schedule resolved: the
// dim-0 carry (smem), an in-group neighbour (smem U of the group), a published / halo trace (staged into
// smem at the group start), or a direct read of the neighbour cell (global).
template <int D, int N, int X, int SX, int SY>
__device__ __forceinline__ void trace_in(const CellParams &p, const CellInfo &ci, int r, int sR, int R, const GroupBufs &gb,
                                         LineSpeed ls, const double *stg, double (&t)[N]) {
  using G = CGeo<D, N>;
  constexpr bool kLean = lean<D, N>();
  switch (ci.src[X]) {
    case kSrcCarry:
      load_vec<N>(gb.carry + N * r, t, false);
      break;
    case kSrcPub:
    case kSrcHalo:
      if constexpr (kLean) load_vec<N>(ci.tsrc[X] + N * r, t, true);
      else load_vec<N>(stg, t, false);
      break;
    case kSrcGroup:
      trace_cell<D, N, X, SX, SY, true>(p, gb.Ugrp + (size_t)ci.nb[X] * G::NDP, sR, ls, ci.sg[X], p.var[X], t);
      break;
    default:
      trace_cell<D, N, X, SX, SY, false>(p, ci.tsrc[X], R, ls, ci.sg[X], p.var[X], t);
      break;
  }
}
// Copy a published / halo trace of dim X (N values at N*r of the trace, L2) into the thread's staging
// slot, asynchronously (issued for every phase at the group start).
template <int N, int X>
__device__ __forceinline__ void stage_trace(const CellInfo &ci, int r, double *stg) {
  if (ci.src[X] != kSrcPub && ci.src[X] != kSrcHalo) return;
  const double *src = ci.tsrc[X] + N * r;
  if constexpr (N % 2 == 0) {
#pragma unroll
    for (int l = 0; l < N; l += 2) cp_async16(stg + l, src + l);
  } else {
#pragma unroll
    for (int l = 0; l < N; ++l) cp_async8(stg + l, src + l);
  }
}
// staging slot of (phase, P|Q) for thread tid: [NPH][2][256 threads][N]
template <int N>
__device__ __forceinline__ double *stg_slot(double *stg, int ph, int q, int tid) {
  return stg + ((size_t)(ph * 2 + q) * 256 + tid) * N;
}
template <int D, int N, int PH>
__device__ __forceinline__ void stage_phase(const CellInfo &ci, int r, double *stg, int tid) {
  using G = CGeo<D, N>;
  stage_trace<N, G::P(PH)>(ci, r, stg_slot<N>(stg, PH, 0, tid));
  if constexpr (G::QA(PH)) stage_trace<N, G::Q(PH)>(ci, r, stg_slot<N>(stg, PH, 1, tid));
  cp_async_commit();
}

// rank-1 lifts of the (scaled) upwind traces: acc[a][b] += lam[a] tP[b] (dim P), acc[a][b] += lam[b] tQ[a]
template <int N, int S>
__device__ __forceinline__ void lift_P(double (&acc)[N][N], const double (&t)[N]) {
#pragma unroll
  for (int b = 0; b < N; ++b)
#pragma unroll
    for (int a = 0; a < N; ++a) acc[a][b] = fma(c_tab[N].lam[S][a], t[b], acc[a][b]);
}
template <int N, int S>
__device__ __forceinline__ void lift_Q(double (&acc)[N][N], const double (&t)[N]) {
#pragma unroll
  for (int a = 0; a < N; ++a)
#pragma unroll
    for (int b = 0; b < N; ++b) acc[a][b] = fma(c_tab[N].lam[S][b], t[a], acc[a][b]);
}

// One phase: tile over (P, Q) at this thread's rest coordinates. Its published traces were staged into
// smem at the group start (cp.async group WAIT = the number of this thread's commits after it).
//  * LAST: `stage_du` (RK) copies the stage's dU into this thread's own (just read) accumulator slots; the
//    next group's cells already stream into the third buffer since the group start, so no barrier here.
//  (was: LAST: after every thread has loaded its tile (barrier), `refill` streams the next group into the
//    accumulator buffer (and RK dU into the thread's own U slots), overlapping the last phase.
template <int D, int N, int MODE, int PH, int WAIT, class Refill>
__device__ __forceinline__ void run_phase(const CellParams &p, const CellInfo &ci, const double *ptab, double *stg, int r,
                                          const GroupBufs &gb, bool active, Refill &&refill,
                                          unsigned long long *pf_sub = nullptr) {
  HD_SUB_DECL
  using G = CGeo<D, N>;
  constexpr bool kLean = lean<D, N>();
  constexpr int P = G::P(PH), Q = G::Q(PH);
  constexpr bool QA = G::QA(PH);
  constexpr int SP = ipow(N, P), SQ = ipow(N, Q);
  constexpr bool FIRST = PH == 0, LAST = PH == G::NPH - 1;
  const Tables1D &T = c_tab[N];
  const int tid = (int)threadIdx.x;

  double uv[N][N], acc[N][N], tP[N], tQ[N];
  LineSpeed lsP{0.0, 0.0}, lsQ{0.0, 0.0};
  int R = 0, sR = 0;
  if (active) {
    // per-thread phase constants (phase_table, once per launch)
    const double *pt = ptab + PH * 1024;
    const int2 rs = reinterpret_cast<const int2 *>(pt + 768)[tid];
    R = rs.x;
    sR = rs.y;
    lsP = line_speed(p, P, Q, ci.base[P], pt[tid]);
    if constexpr (QA) lsQ = line_speed(p, Q, P, ci.base[Q], pt[256 + tid]);
    if constexpr (P == 0 && N % 2 == 0) {
#pragma unroll
      for (int b = 0; b < N; ++b)
#pragma unroll
        for (int a = 0; a < N; a += 2) {
          const double2 v = *reinterpret_cast<const double2 *>(gb.U + sidx<D, N>(sR, a + b * SQ));
          uv[a][b] = v.x;
          uv[a + 1][b] = v.y;
        }
    } else {
#pragma unroll
      for (int a = 0; a < N; ++a)
#pragma unroll
        for (int b = 0; b < N; ++b) uv[a][b] = gb.U[sidx<D, N>(sR, a * SP + b * SQ)];
    }
    if constexpr (!FIRST && !kLean) {
#pragma unroll
      for (int a = 0; a < N; ++a)
#pragma unroll
        for (int b = 0; b < N; ++b) acc[a][b] = gb.A[sidx<D, N>(sR, a * SP + b * SQ)];
    }
  }
  // volume terms of P and Q and this cell's downwind traces along P and Q (stored right away)
  // lean: one carry buffer -- the incoming dim-0 carry (this thread's own slot) is read before the pass
  // overwrites it with the outgoing one; the passes start a fresh accumulator (the earlier phases' sum is
  // added after the lifts), so the tile and the old accumulator are never live together
  constexpr bool EARLY = kLean && P == 0;
  auto passes = [&]() {
    if constexpr (EARLY) trace_in<D, N, P, SP, SQ>(p, ci, r, sR, R, gb, lsP, stg_slot<N>(stg, PH, 0, tid), tP);
    {
      double tr[N];
      pass_P_any<N, P, FIRST || kLean>(p, acc, uv, lsP, tr, ci.sg[P], p.var[P]);
      const unsigned char oP = ci.out[P];
      if (oP == kOutCarry) store_vec<N>(gb.carry_out + N * r, tr, false);
      else if (oP == kOutPub) {
        // slab super-units: the dim-1 trace is read by this CTA one slab row later -- keep it in L2
        bool kept = false;
        if constexpr (P == 1 && kLean && N % 2 == 0) {
          if (p.slab > 1) {
            store_vec_keep<N>(p.tbuf[P] + (size_t)ci.oslot * G::FN + (size_t)N * r, tr);
            kept = true;
          }
        }
        if (!kept) store_vec<N>(p.tbuf[P] + (size_t)ci.oslot * G::FN + (size_t)N * r, tr, true);
      }
    }
    if constexpr (QA) {
      double tr[N];
      pass_Q_any<N, Q>(p, acc, uv, lsQ, tr, ci.sg[Q], p.var[Q]);
      if (ci.out[Q] == kOutPub) store_vec<N>(p.tbuf[Q] + (size_t)ci.oslot * G::FN + (size_t)N * r, tr, true);
    }
  };
  // lean, last phase: the next group's fill (refill: barrier + cp.async into the U buffer, reached by every
  // thread) comes after the epilogue -- RK re-reads U there (U' = U + B_s dU), and in A mode issuing it
  // after the passes kept the accumulator live across the fill code (spills; measured 4-9% slower)
  if constexpr (kLean) {
    if (active) passes();
  } else {
    if constexpr (LAST) refill(sR, R);  // RK: dU into this thread's own accumulator slots (read above)
    if (!active) return;
    passes();
  }
  if (active) {
  const size_t g0 = (size_t)ci.cell * G::ND + R;
  HD_SUB(2);
  // upwind traces (the staged ones have arrived once this thread's copies of this phase are complete)
  if constexpr (!kLean) cp_async_wait<WAIT>();
  if constexpr (!EARLY) trace_in<D, N, P, SP, SQ>(p, ci, r, sR, R, gb, lsP, stg_slot<N>(stg, PH, 0, tid), tP);
  if (ci.sg[P]) lift_P<N, 1>(acc, tP);
  else lift_P<N, 0>(acc, tP);
  if constexpr (kLean && P == 1 && N == 4 && D >= 5) {
    // slab super-units: a consumed dim-1 trace has no other reader -- once the warp's lifts used every lane's
    // values, drop its lines from L2 without a write-back (one lane per 128-byte line of 4 threads' traces)
    if (p.slab > 1 && ci.src[1] == kSrcPub) {
      __syncwarp();
      if ((tid & 3) == 0) discard_l2(ci.tsrc[1] + N * r);
    }
  }
  HD_SUB(3);
  if constexpr (QA) {
    trace_in<D, N, Q, SQ, SP>(p, ci, r, sR, R, gb, lsQ, stg_slot<N>(stg, PH, 1, tid), tQ);
    if (ci.sg[Q]) lift_Q<N, 1>(acc, tQ);
    else lift_Q<N, 0>(acc, tQ);
  }
  if constexpr (kLean && !FIRST) {
#pragma unroll
    for (int a = 0; a < N; ++a)
#pragma unroll
      for (int b = 0; b < N; ++b) acc[a][b] += gb.A[sidx<D, N>(sR, a * SP + b * SQ)];
  }
  HD_SUB(4);

  if constexpr (!LAST && P == 0 && N % 2 == 0) {
#pragma unroll
    for (int b = 0; b < N; ++b)
#pragma unroll
      for (int a = 0; a < N; a += 2)
        *reinterpret_cast<double2 *>(gb.A + sidx<D, N>(sR, a + b * SQ)) = make_double2(acc[a][b], acc[a + 1][b]);
  } else if constexpr (!LAST) {
#pragma unroll
    for (int a = 0; a < N; ++a)
#pragma unroll
      for (int b = 0; b < N; ++b) gb.A[sidx<D, N>(sR, a * SP + b * SQ)] = acc[a][b];
  } else if constexpr (MODE == kModeAdvection || MODE == kModeAdvAcc) {
    // weak form: v = M (M^-1 A u), M_qq = |J| prod_i w_{q_i}; kModeAdvAcc (second one-sided half of a
    // central-flux application) adds to v
    const double wr = ptab[PH * 1024 + 512 + tid];
#pragma unroll
    for (int a = 0; a < N; ++a)
#pragma unroll
      for (int b = 0; b < N; ++b) {
        double v = acc[a][b] * (wr * (T.w[a] * T.w[b]));
        if constexpr (MODE == kModeAdvAcc) v += __ldcs(p.out + g0 + a * SP + b * SQ);
        __stcs(p.out + g0 + a * SP + b * SQ, v);
      }
  } else {
    // LSRK 2N stage: dU <- A_s dU + dt M^-1 A(U); U_new <- U + B_s dU. U is still in uv; dU arrived
    // (cp.async issued by stage_du) in this thread's own slots of the accumulator buffer.
    if constexpr (MODE == kModeRK && kLean) {
      // lean: dU straight from L2 (prefetched at the group start)
#pragma unroll
      for (int a = 0; a < N; ++a)
#pragma unroll
        for (int b = 0; b < N; ++b) acc[a][b] = fma(p.rk_a, __ldcs(p.du + g0 + a * SP + b * SQ), acc[a][b]);
    } else if constexpr (MODE == kModeRK) {
      cp_async_wait<0>();
#pragma unroll
      for (int a = 0; a < N; ++a)
#pragma unroll
        for (int b = 0; b < N; ++b) acc[a][b] = fma(p.rk_a, gb.A[sidx<D, N>(sR, a * SP + b * SQ)], acc[a][b]);
    }
#pragma unroll
    for (int a = 0; a < N; ++a)
#pragma unroll
      for (int b = 0; b < N; ++b) {
        __stcs(p.du + g0 + a * SP + b * SQ, acc[a][b]);
        // lean: U re-read from the U buffer instead of keeping the tile live
        const double u0 = kLean ? gb.U[sidx<D, N>(sR, a * SP + b * SQ)] : uv[a][b];
        __stcs(p.out + g0 + a * SP + b * SQ, fma(p.rk_b, acc[a][b], u0));
      }
  }
  HD_SUB(5);
  }  // active
  if constexpr (LAST && kLean) refill(sR, R);  // every thread, after its U-buffer reads
}

// Shared-memory carve-up (offsets in doubles, every region 16-byte aligned):
// bufs[3][CT*NDP] (two cell buffers alternating, one accumulator) | carry[2][CT*FN] | ptab[NPH][1024] |
// stg[NPH][2][256][N] | info[2][CT] | raw[4][CT*D] | rawc[4][CT] (the schedule-record ring) | uq[8] (unit
// queue). Lean kernel: bufs[2] (U, accumulator), carry[1], no stg.
__host__ __device__ constexpr int round2(int x) { return (x + 1) & ~1; }
template <int D, int N>
struct SmemMap {
  int carry, ptab, stg, info, raw, rawc, uq, bytes;
  __host__ __device__ constexpr SmemMap(int CT)
      : carry(0), ptab(0), stg(0), info(0), raw(0), rawc(0), uq(0), bytes(0) {
    using G = CGeo<D, N>;
    constexpr bool kLean = lean<D, N>();
    carry = round2((kLean ? 2 : 3) * CT * G::NDP);
    ptab = carry + round2((kLean ? 1 : 2) * CT * G::FN);
    stg = ptab + G::NPH * 1024;
    info = stg + (kLean ? 0 : round2(G::NPH * 2 * 256 * N));
    raw = info + round2(2 * CT * (int)sizeof(CellInfo) / 8);
    rawc = raw + 4 * CT * D * (int)sizeof(SchedDim) / 8;
    uq = rawc + round2(4 * CT * (int)sizeof(SchedCell) / 8);
    bytes = (uq + 4) * 8;
  }
};
static_assert(sizeof(CellInfo) % 8 == 0 && sizeof(SchedDim) % 16 == 0 && sizeof(SchedCell) == 8, "smem records");
// Largest group (cells) the kernel lays out: every smem offset is a compile-time constant for it (a mesh
// with a smaller group leaves part of the buffers unused).
template <int D, int N>
__host__ __device__ constexpr int max_ct() {
  int c = 256 / CGeo<D, N>::NT;
  while (c > 1 && SmemMap<D, N>(c).bytes > 227 * 1024) --c;
  return c;
}
template <int D, int N>
__host__ __device__ constexpr int cell_smem_bytes() {
  return SmemMap<D, N>(max_ct<D, N>()).bytes;
}

// Persistent kernel: CTA b processes units u_begin + b, + grid, ... < u_end in increasing order (the whole
// mesh, or one v-chunk of a pipelined multi-rank stage); each unit is GPU groups.
// Per group: the next group's schedule records are staged (cp.async) at the start, its producers' flags
// read (ld.acquire) one phase later and resolved after the epilogue; its cells stream into the free buffer
// during the last phase. The progress flag of a group is released (st.release after a CTA barrier) at
// the next group's start.
template <int D, int N, int MODE>
__global__ void __launch_bounds__(256, lean<D, N>() ? 2 : 1) cell_kernel(const __grid_constant__ CellParams p) {
  using G = CGeo<D, N>;
  constexpr bool kLean = lean<D, N>();
  constexpr int NPH = G::NPH;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int CT = p.CT;
  constexpr int MAXCT = max_ct<D, N>();
  constexpr int CND = MAXCT * G::NDP;
  double *smem = reinterpret_cast<double *>(smem_raw);
  constexpr SmemMap<D, N> map(MAXCT);
  double *bufs = smem;
  double *carry0 = smem + map.carry;
  double *ptab = smem + map.ptab;
  double *stg = smem + map.stg;
  CellInfo *info0 = reinterpret_cast<CellInfo *>(smem + map.info);
  SchedDim *raw = reinterpret_cast<SchedDim *>(smem + map.raw);
  SchedCell *rawc = reinterpret_cast<SchedCell *>(smem + map.rawc);
  const int tid = threadIdx.x;
  const int nthr = (int)blockDim.x;
  const int k = tid / G::NT;
  const int r = tid - k * G::NT;
  const bool active = k < CT;
  const int kk0 = active ? k : 0;
  if (p.u_begin + (int)blockIdx.x >= p.u_end) return;
  phase_table<D, N, MODE>(p, r, ptab);  // read only by this thread
  const int nitems = CT * D;

  // the group's cells: CT cells at cell stride cstride into the padded layout, 16-byte cp.async per pair
  // of dim-0 neighbours. Fast path (N = 4, 256 threads, CT n^d a multiple of 512): thread tid copies the
  // pairs x = 2 tid + 512 j, whose smem position is additive in (tid, j) -- swz(2 tid mod n^d) once per
  // launch plus a compile-time offset (no digit carries between the two parts for N = 4).
  constexpr bool FASTFILL = N == 4 && G::NT * MAXCT == 256 && (G::ND % 512 == 0 || 512 % G::ND == 0);
  const int fbase = swz<D, N>((2 * tid) % G::ND);
  const int fcell0 = (2 * tid) / G::ND;
  const unsigned long long pol_ef = HD_FILL_EF ? l2_policy_evict_first() : 0ull;
  auto copy_cells = [&](int first_cell, double *dst) {
    HD_DCHECK(p, first_cell >= 0 && first_cell + (CT - 1) * p.cstride < p.ncells, 1);
    if constexpr (FASTFILL) {
      if (nthr == 256 && (CT * G::ND) % 512 == 0) {
        if constexpr (G::ND >= 512) {
          for (int kc = 0; kc < CT; ++kc) {
            const double *src = p.u + ((size_t)first_cell + kc * p.cstride) * G::ND + 2 * tid;
            double *d0 = dst + kc * G::NDP + fbase;
#pragma unroll
            for (int m = 0; m < G::ND / 512; ++m) {
              if constexpr (HD_FILL_EF) cp_async16_hint(d0 + swz<D, N>(512 * m), src + 512 * m, pol_ef);
              else cp_async16(d0 + swz<D, N>(512 * m), src + 512 * m);
            }
          }
        } else {
          for (int j = 0; j < CT * G::ND / 512; ++j) {
            const int kc = j * (512 / G::ND) + fcell0;
            cp_async16(dst + kc * G::NDP + fbase, p.u + ((size_t)first_cell + kc * p.cstride) * G::ND + (2 * tid) % G::ND);
          }
        }
        return;
      }
    }
    if constexpr (G::ND % 2 == 0) {
      for (int i = tid; i < ((CT * G::ND) >> 1); i += nthr) {
        const int e = 2 * i, kc = e / G::ND, x = e - kc * G::ND;
        cp_async16(dst + kc * G::NDP + swz<D, N>(x), p.u + ((size_t)first_cell + kc * p.cstride) * G::ND + x);
      }
    } else {
      for (int i = tid; i < CT * G::ND; i += nthr) {
        const int kc = i / G::ND, x = i - kc * G::ND;
        cp_async8(dst + kc * G::NDP + swz<D, N>(x), p.u + ((size_t)first_cell + kc * p.cstride) * G::ND + x);
      }
    }
  };
  // Schedule records: a ring of kRing groups in smem, fetched (cp.async, spread over the threads) three
  // groups ahead of their use, so no thread waits for them. The (cell, dim) items of a group -- flag
  // acquire and resolution into CellInfo -- are spread over the warps (lane j of warp w: item j*nwarps + w),
  // so no warp carries the group's bookkeeping alone.
  constexpr int kRing = 4;
  auto fetch = [&](int slot, long long gs) {
    const char *src = reinterpret_cast<const char *>(p.sched + gs * nitems);
    char *dst = reinterpret_cast<char *>(raw + slot * MAXCT * D);
    for (int q = tid; q < nitems * 2; q += nthr) cp_async16(dst + 16 * q, src + 16 * q);
    for (int q = tid; q < CT; q += nthr) cp_async8(rawc + slot * MAXCT + q, p.schedc + gs * CT + q);
  };
  // the CTA's group sequence: iteration it -> (unit, step); j groups ahead of (u0, g0). Dynamic dealing
  // (HD_DYN): after its first unit (u_begin + blockIdx) a CTA takes the next unit from the launch's counter;
  // the units it will run are queued in smem (uq[k & 7] = its k-th unit, qk = the current one), grabbed by
  // one thread a group before anybody reads them. Units still start in increasing order, so the published-
  // trace protocol is unchanged, and a CTA that runs slower than its SM neighbour takes fewer units.
  int *uq = reinterpret_cast<int *>(smem + map.uq);
  int qk = 0, ngrab = 1;
  auto ahead = [&](int u0, int g0, int j, int &uo, int &go) {
    uo = u0;
    go = g0 + j;
    if constexpr (kDyn) {
      int k = qk;
      while (go >= p.GPU) {
        go -= p.GPU;
        ++k;
      }
      if (k != qk) uo = uq[k & 7];
    } else {
      while (go >= p.GPU) {
        go -= p.GPU;
        uo += gridDim.x;
      }
    }
    return uo < p.u_end;
  };
  auto grab_upto = [&](int kneed) {  // one thread: queue the units up to the kneed-th
    while (ngrab <= kneed) {
      uq[ngrab & 7] = p.u_begin + (int)gridDim.x + atomicAdd(p.uctr, 1);
      ++ngrab;
    }
  };
  const int nwarps = nthr >> 5;
  const int item0 = nitems <= nthr ? (tid & 31) * nwarps + (tid >> 5) : tid;
  int fv0 = 0, fv1 = 0;  // producer flag values of this thread's items (at most 2 items per thread)
  auto acquire = [&](int slot) {
    const SchedDim *rs = raw + slot * MAXCT * D;
    int j = 0;
    for (int idx = item0; idx < nitems; idx += nthr, ++j) {
      const SchedDim &rr = rs[idx];
      if (rr.src == kSrcPub) {
        const int v = ld_acquire(p.flags + rr.pflag);
        if (j == 0) fv0 = v;
        else fv1 = v;
      } else if (rr.src == kSrcDirect && p.prefetch && HD_PF_DIRECT == 1) {
        prefetch_l2(p.u + (size_t)rr.nb * p.ND, (unsigned)(p.ND * 8));
      }
    }
  };
  auto resolve = [&](int slot, CellInfo *inf) {
    const SchedDim *rs = raw + slot * MAXCT * D;
    const SchedCell *rc = rawc + slot * MAXCT;
    int j = 0;
    for (int idx = item0; idx < nitems; idx += nthr, ++j) {
      const int kc = idx / D, i = idx - kc * D;
      const SchedDim &rr = rs[idx];
      CellInfo &ci = inf[kc];
      unsigned char src = rr.src;
      const double *ts = nullptr;
      if (src == kSrcPub) {
        // flags read in phase 1 (acquire); a producer that was not done then gets a second look now, two
        // phases later -- a producer running only slightly behind its nominal lead is then usually done
        int fv = j == 0 ? fv0 : fv1;
        if (fv < (p.epoch | rr.need)) fv = ld_acquire(p.flags + rr.pflag);
        if (fv >= (p.epoch | rr.need)) {
          ts = p.tbuf[i] + (size_t)rr.slot * p.FN;
          // the whole trace into L2 now, a group before the phase reads it (+5% 6D)
          if (HD_PF_PUB && p.prefetch) prefetch_l2(ts, (unsigned)(p.FN * 8));
        } else {
          src = kSrcDirect;  // not published yet: read the neighbour cell itself
          if (p.prefetch) prefetch_l2(p.u + (size_t)rr.nb * p.ND, (unsigned)(p.ND * 8));
        }
      } else if (src == kSrcHalo) {
        ts = p.hbuf[i] + (size_t)rr.slot * p.FN;
        if (HD_PF_PUB && p.prefetch) prefetch_l2(ts, (unsigned)(p.FN * 8));
      }
      if (src == kSrcDirect) ts = p.u + (size_t)rr.nb * p.ND;
      if (HD_PF_DIRECT == 2 && rr.src == kSrcDirect && p.prefetch) prefetch_l2(ts, (unsigned)(p.ND * 8));
#ifdef HD_COUNT
      if (rr.src == kSrcPub) atomicAdd(p.err + (src == kSrcPub ? 25 : 26), 1);
      else if (src == kSrcDirect) atomicAdd(p.err + 27, 1);
#endif
      HD_DCHECK(p, rc[kc].cell >= 0 && rc[kc].cell < p.ncells && rr.nb >= 0 && rr.nb < p.ncells, 1);
      HD_DCHECK(p, src != kSrcPub || (rr.slot >= 0 && rr.slot < p.ncells && rr.pflag >= 0 && rr.pflag < p.nunits), 1);
      HD_DCHECK(p, src != kSrcGroup || (rr.slot >= 0 && rr.slot < CT), 1);
      HD_DCHECK(p, src != kSrcHalo || (rr.slot >= 0 && rr.slot < p.nhalo[i]), 1);
      HD_DCHECK(p, src != kSrcHalo || p.rtag[i * 2 + rr.sg] == p.epoch, 2);  // halo of this stage
      ci.base[i] = rr.base;
      ci.tsrc[i] = ts;
      ci.nb[i] = (unsigned char)rr.slot;
      ci.src[i] = src;
      ci.out[i] = rr.out;
      ci.sg[i] = rr.sg;
      if (i == 0) {
        ci.cell = rc[kc].cell;
        ci.oslot = rc[kc].oslot;
      }
    }
  };

  int u = p.u_begin + (int)blockIdx.x, gi = 0, it = 0;
  if constexpr (kDyn) {
    if (tid == nthr - 1) {
      uq[0] = u;
      grab_upto(4 / p.GPU);
    }
    __syncthreads();
  }
  // prologue: the records of the first three groups, group 0's schedule and cells
  for (int j = 0; j < kRing - 1; ++j) {
    int ua, ga;
    if (ahead(u, gi, j, ua, ga)) fetch(j, (long long)ua * p.GPU + ga);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  acquire(0);
  resolve(0, info0);
  copy_cells(rawc[0].cell, bufs);
  cp_async_commit();
  cp_async_wait<0>();
  int prev_unit = -1, prev_step = 0;
  HD_PROF_DECL
  while (u < p.u_end) {
    const int s = it & 1;
    const int slot1 = (it + 1) % kRing;  // records of the next group
    int un, gn;
    const bool has_next = ahead(u, gi, 1, un, gn);
    // group g-1 done (its traces written, its epilogue finished); this group's cells and info are in smem
    HD_PROF_BAR(0);
    HD_PROF_GROUP();
    if (prev_unit >= 0 && tid == nthr - 1) st_release(p.flags + prev_unit, p.epoch | (prev_step + 1));
    // the units the next group's lookahead reaches (read after the next barrier)
    if (kDyn && tid == nthr - 1) grab_upto(qk + (gi + 4) / p.GPU);
    const CellInfo &ci = info0[s * MAXCT + kk0];
    GroupBufs gb;
    gb.Ugrp = bufs + (kLean ? 0 : s) * CND;
    gb.U = gb.Ugrp + (size_t)kk0 * G::NDP;
    gb.A = bufs + (kLean ? 1 : 2) * CND + (size_t)kk0 * G::NDP;
    gb.carry = carry0 + (size_t)((kLean ? 0 : s) * MAXCT + kk0) * G::FN;
    gb.carry_out = carry0 + (size_t)((kLean ? 0 : s ^ 1) * MAXCT + kk0) * G::FN;
    // cp.async groups of this thread, in commit order: this group's staged traces per phase, the records of
    // the group three ahead, then (last phase) RK dU and the next group's cells
    if constexpr (kLean) {
    } else if (active) {
      stage_phase<D, N, 0>(ci, r, stg, tid);
      if constexpr (NPH > 1) stage_phase<D, N, (NPH > 1 ? 1 : 0)>(ci, r, stg, tid);
      if constexpr (NPH > 2) stage_phase<D, N, (NPH > 2 ? 2 : 0)>(ci, r, stg, tid);
    } else {
      for (int q = 0; q < NPH; ++q) cp_async_commit();
    }
    HD_MARK(0);
    {
      int ua, ga;
      if (ahead(u, gi, kRing - 1, ua, ga)) fetch((it + kRing - 1) % kRing, (long long)ua * p.GPU + ga);
      cp_async_commit();
    }
    if (!kLean && MODE == kModeRK && tid == 0 && p.prefetch)
      for (int kc = 0; kc < CT; ++kc)
        prefetch_l2(p.du + ((size_t)info0[s * MAXCT].cell + kc * p.cstride) * G::ND, (unsigned)(G::ND * 8));
    HD_MARK(1);
    auto flags_next = [&]() {
      if (has_next) {
        acquire(slot1);
        // the cells of the group after next into L2 (its fill is issued at the next group's start); lean: the
        // next group's (its fill is issued in this group's last phase) -- with two CTAs per SM a group takes
        // twice as long, and two groups of HBM traffic would cycle the whole L2 before the fill
        int ua, ga;
        constexpr int kAhead = kLean ? HD_LEAN_PF : 2;
        if (tid == 0 && p.prefetch && kAhead > 0 && ahead(u, gi, kAhead, ua, ga)) {
          const int slot2 = (it + kAhead) % kRing;
          for (int kc = 0; kc < CT; ++kc)
            prefetch_l2(p.u + ((size_t)rawc[slot2 * MAXCT].cell + kc * p.cstride) * G::ND, (unsigned)(G::ND * 8));
        }
      }
      // lean RK: this group's dU into L2 for the epilogue's direct reads
      if (kLean && MODE == kModeRK && tid == 32 && p.prefetch && HD_PF_DU == 1)
        for (int kc = 0; kc < CT; ++kc)
          prefetch_l2(p.du + ((size_t)info0[s * MAXCT].cell + kc * p.cstride) * G::ND, (unsigned)(G::ND * 8));
    };
    // the next group's cells stream into the other cell buffer (free since the previous group ended)
    if constexpr (!kLean) {
      if (has_next) copy_cells(rawc[slot1 * MAXCT].cell, bufs + (s ^ 1) * CND);
      cp_async_commit();
    }
    HD_MARK(2);
    auto refill = [&](int sR, int R) {
      // RK: dU of this thread's tile into its own (already read) accumulator slots
      if constexpr (MODE == kModeRK && !kLean) {
        if (active) {
          constexpr int P = G::P(NPH - 1), Q = G::Q(NPH - 1);
          constexpr int SP = ipow(N, P), SQ = ipow(N, Q);
          const double *src = p.du + (size_t)ci.cell * G::ND + R;
#pragma unroll
          for (int a = 0; a < N; ++a)
#pragma unroll
            for (int b = 0; b < N; ++b) cp_async8(gb.A + sidx<D, N>(sR, a * SP + b * SQ), src + a * SP + b * SQ);
        }
        cp_async_commit();
      }
      if constexpr (kLean) {
        // every thread has read its last-phase tiles: the next group's cells stream into the U buffer
        __syncthreads();
        if (has_next) copy_cells(rawc[slot1 * MAXCT].cell, bufs);
        cp_async_commit();
      }
    };
    auto none = [](int, int) {};
    // pending commits after phase PH's traces when its lifts wait: the later phases' traces, the records
    // and the next group's cells; in the last phase the records, the cells and (RK) dU
    constexpr int WLAST = 2 + (MODE == kModeRK ? 1 : 0);
    if constexpr (NPH == 1) {
      flags_next();
      run_phase<D, N, MODE, 0, WLAST>(p, ci, ptab, stg, r, gb, active, refill);
    } else {
      run_phase<D, N, MODE, 0, NPH + 1>(p, ci, ptab, stg, r, gb, active, none, HD_PF(0));
      HD_MARK(3);
      HD_PROF_BAR(1);
      flags_next();
      HD_MARK(4);
      if constexpr (NPH == 2) {
        run_phase<D, N, MODE, (NPH > 1 ? 1 : 0), WLAST>(p, ci, ptab, stg, r, gb, active, refill);
      } else {
        run_phase<D, N, MODE, (NPH > 1 ? 1 : 0), 3>(p, ci, ptab, stg, r, gb, active, none, HD_PF(1));
        HD_MARK(5);
        HD_PROF_BAR(2);
        if (kLean && MODE == kModeRK && tid == 32 && p.prefetch && HD_PF_DU == 2)
          for (int kc = 0; kc < CT; ++kc)
            prefetch_l2(p.du + ((size_t)info0[s * MAXCT].cell + kc * p.cstride) * G::ND, (unsigned)(G::ND * 8));
        run_phase<D, N, MODE, (NPH > 2 ? 2 : 0), WLAST>(p, ci, ptab, stg, r, gb, active, refill, HD_PF(2));
        HD_MARK(6);
      }
    }
    if (has_next) resolve(slot1, info0 + (s ^ 1) * MAXCT);
    HD_MARK(7);
    cp_async_wait<0>();  // the next group's cells (and the records fetched this group)
    prev_unit = p.flags ? u : -1;
    prev_step = gi;
    if (gi + 1 >= p.GPU) ++qk;
    u = un;
    gi = gn;
    ++it;
  }
  if (prev_unit >= 0) {
    __syncthreads();
    if (tid == nthr - 1) st_release(p.flags + prev_unit, p.epoch | (prev_step + 1));
  }
  HD_PROF_DUMP();
}

}  // namespace hd
