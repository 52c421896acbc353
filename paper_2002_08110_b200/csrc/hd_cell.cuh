// hd_cell.cuh -- the fused cell kernel (element-centric loop, Alg. 1/Alg. 2) for sm_100a.
// Included by hd_kernels.cu (single translation unit with the __constant__ tables).
//
// One CTA iteration processes one work item = C consecutive cells along dim 0 (C | L_0). Items are
// visited in lexicographic item order, with the direction of every "trace" dimension (a dimension
// whose speed has one sign on the whole box) reversed when that sign is negative, so the upwind
// neighbour along a trace dim is always processed istride_i items earlier (except at the periodic
// wrap). Each thread owns, per phase, an n x n tile of a cell over two dimensions (P, Q) at fixed
// other coordinates (its "rest" index r):
//   1. read the lines of its tile from smem (the item was gathered with cp.async into a padded
//      layout, prefetched one item ahead) and form, line by line, the volume terms of P and Q (1D
//      matrices with the own-face term folded in) and the cell's DOWNWIND traces along P and Q,
//   2. publish those traces (ring / full-size buffer) and bump the item's per-phase flag (one
//      release per warp),
//   3. obtain the UPWIND traces: acquire the producer item's flag and read n values per dim (tried
//      early, before step 1, when the producer is long done); at the periodic wrap and for dims
//      whose speed changes sign, form them from the neighbour cell itself (L1/L2 reads),
//   4. add the rank-1 lifts, then hand the accumulator to the next phase through smem, or finish:
//      weak-form scaling by the collocated mass (A mode) or the LSRK 2N update (RK mode).
#pragma once

#ifndef HD_EARLY_TRACES
#define HD_EARLY_TRACES 0
#endif
#ifndef HD_PUBLISH_FENCE
#define HD_PUBLISH_FENCE 0
#endif
#ifndef HD_DU_DIRECT
#define HD_DU_DIRECT 0
#endif

namespace hd {

template <int D, int N>
struct CGeo {
  static constexpr int ND = ipow(N, D);
  static constexpr int FN = ipow(N, D - 1);   // face points per face
  static constexpr int NT = ipow(N, D - 2);   // threads per cell
  static constexpr int NPH = (D + 1) / 2;     // phases
  static constexpr __host__ __device__ int P(int ph) { return (D % 2 == 1 && ph == NPH - 1) ? D - 1 : 2 * ph; }
  static constexpr __host__ __device__ int Q(int ph) { return (D % 2 == 1 && ph == NPH - 1) ? D - 2 : 2 * ph + 1; }
  static constexpr __host__ __device__ bool QA(int ph) { return !(D % 2 == 1 && ph == NPH - 1); }
  // one cell must fit three padded smem buffers (2 CTAs per SM up to 110 KB, else 1 CTA per SM)
  static constexpr bool OK = NT <= 256 && ND * 8 * 9 / 8 * 3 + 4096 <= 220 * 1024;
};

// padded smem layout: 2 doubles of padding after every 16 (conflict-free row access)
__host__ __device__ constexpr int padded(int e) { return e + ((e >> 4) << 1); }

struct CellInfo {
  int cell;                 // local memory index of the cell
  int c[kMaxD];             // cell coordinates
  int t[kMaxD];             // traversal coordinates (item level for dim 0)
  int sg[kMaxD];            // 1: a_i < 0 on this cell (upwind neighbour at +e_i)
  int direct[kMaxD];        // 1: form the upwind trace from the neighbour cell itself
  int nbcell[kMaxD];        // local memory index of the upwind neighbour
  int pitem[kMaxD];         // producer item of the upwind trace
  int pk[kMaxD];            // producer cell slot in that item
  double base[kMaxD];       // a_i at the cell's lower corner: a_const + sum_j a_lin[i][j] (lo_j + c_j h_j)
};

// per-thread, per-phase constants
struct ThreadPhase {
  double wP, wQ;            // sum over rest dims j of a_lin[P|Q][j] h_j xi_{m_j}
  double wr;                // |J| prod_{rest j} w_{m_j} (weak-form mass of the last phase)
  int R;                    // cell-local offset of the rest coordinates
  int pad;
};

__device__ __forceinline__ int ld_acquire(const int *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Release increment of a publication counter. Issued by one lane after __syncwarp(): the warp
// barrier orders the other lanes' trace stores before it, and release makes them visible to any
// thread that acquires the counter.
__device__ __forceinline__ void red_release_add(int *p) {
#if HD_PUBLISH_FENCE
  __threadfence();
  atomicAdd(p, 1);
#else
  asm volatile("red.release.gpu.global.add.s32 [%0], 1;\n" ::"l"(p) : "memory");
#endif
}
// Spin until a producer flag reaches the target. A watchdog aborts the kernel (trap) instead of
// hanging if a publication never arrives (a protocol bug would otherwise wedge the GPU).
__device__ __forceinline__ void wait_flag(const int *p, int target) {
  if (ld_acquire(p) >= target) return;
  unsigned spins = 0;
  while (ld_acquire(p) < target) {
    __nanosleep(32);
    if (++spins > (1u << 25)) __trap();
  }
}

// Decode item b: all cells' coordinates, upwind neighbours and trace producers. Two steps, each
// spread over the CTA's threads ((cell, dim) pairs); the caller separates them with a barrier.
template <int D>
__device__ __forceinline__ void decode_coords(const CellParams &p, int b, int C, CellInfo *info) {
  for (int idx = threadIdx.x; idx < C * D; idx += blockDim.x) {
    const int k = idx / D, i = idx - k * D;
    const int t = (b / p.istride[i]) % p.IL[i];
    int c = p.dirneg[i] ? p.IL[i] - 1 - t : t;
    if (i == 0) c = c * C + k;
    info[k].t[i] = t;
    info[k].c[i] = c;
  }
}
template <int D>
__device__ __forceinline__ void decode_links(const CellParams &p, int b, int C, CellInfo *info) {
  for (int idx = threadIdx.x; idx < C * D; idx += blockDim.x) {
    const int k = idx / D, i = idx - k * D;
    CellInfo &ci = info[k];
    int cell = 0;
    double ab = p.a_const[i], half = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      cell += ci.c[j] * p.lstride[j];
      ab = fma(p.a_lin[i][j], p.lo[j] + (double)ci.c[j] * p.h[j], ab);
      half = fma(p.a_lin[i][j], 0.5 * p.h[j], half);
    }
    const int sg = (ab + half) < 0.0 ? 1 : 0;  // sign at the cell centre (constant on the cell)
    const int up = sg ? 1 : -1;                // offset of the upwind neighbour along i
    int cn = ci.c[i] + up;
    if (cn < 0) cn += p.L[i];
    if (cn >= p.L[i]) cn -= p.L[i];
    ci.base[i] = ab;
    ci.sg[i] = sg;
    ci.nbcell[i] = cell + (cn - ci.c[i]) * p.lstride[i];
    int direct = 1, pitem = 0, pk = 0;
    if (p.tmode[i] != kTraceNone) {
      if (i == 0 && k + up >= 0 && k + up < C) {
        direct = 0;
        pitem = b;
        pk = k + up;
      } else if (ci.t[i] > 0) {
        direct = 0;
        pitem = b - p.istride[i];
        pk = i == 0 ? (up < 0 ? C - 1 : 0) : k;
      }
    }
    ci.direct[i] = direct;
    ci.pitem[i] = pitem;
    ci.pk[i] = pk;
    if (i == 0) ci.cell = cell;
  }
}

// first cell (in memory) of item b
template <int D>
__device__ __forceinline__ int item_first_cell(const CellParams &p, int b, int C) {
  int cell = 0;
#pragma unroll
  for (int i = 0; i < D; ++i) {
    const int t = (b / p.istride[i]) % p.IL[i];
    int c = p.dirneg[i] ? p.IL[i] - 1 - t : t;
    if (i == 0) c *= C;
    cell += c * p.lstride[i];
  }
  return cell;
}

// Per-thread phase constants for rest index r. sx, sw: the 1D nodes and weights staged in smem.
template <int D, int N, int PH, bool MASS>
__device__ __forceinline__ void thread_phase(const CellParams &p, int r, const double *sx, const double *sw,
                                             ThreadPhase &tp) {
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
      if (p.a_lin[P][j] != 0.0) wP = fma(p.a_lin[P][j] * p.h[j], sx[m], wP);
      if (p.a_lin[Q][j] != 0.0) wQ = fma(p.a_lin[Q][j] * p.h[j], sx[m], wQ);
      if constexpr (MASS) wr *= sw[m];
    }
    nj *= N;
  }
  tp.wP = wP;
  tp.wQ = wQ;
  tp.wr = wr;
  tp.R = R;
  tp.pad = 0;
}

template <int N, int S>
__device__ __forceinline__ void lift_P(double (&acc)[N][N], const double (&st)[N]) {
  const Tables1D &T = c_tab[N];
#pragma unroll
  for (int b = 0; b < N; ++b)
#pragma unroll
    for (int a = 0; a < N; ++a) acc[a][b] = fma(T.lam[S][a], st[b], acc[a][b]);
}
template <int N, int S>
__device__ __forceinline__ void lift_Q(double (&acc)[N][N], const double (&st)[N]) {
  const Tables1D &T = c_tab[N];
#pragma unroll
  for (int a = 0; a < N; ++a)
#pragma unroll
    for (int b = 0; b < N; ++b) acc[a][b] = fma(T.lam[S][b], st[a], acc[a][b]);
}

// smem element address of tile element at logical eb + off in the padded layout; off is a
// compile-time constant after unrolling, so the branches fold away
template <bool EB16>
__device__ __forceinline__ int paddr(int off, int eb, int peb) {
  if ((off & 15) == 0) return peb + off + ((off >> 4) << 1);
  if (EB16 && off < 16) return peb + off;
  return padded(eb + off);
}

template <int N, int SP, int SQ, bool EB16>
__device__ __forceinline__ void load_tile(const double *S, int eb, double (&v)[N][N]) {
  const int peb = padded(eb);
#pragma unroll
  for (int a = 0; a < N; ++a)
#pragma unroll
    for (int b = 0; b < N; ++b) v[a][b] = S[paddr<EB16>(a * SP + b * SQ, eb, peb)];
}

// store / load the n values t[0..n) contiguously (16-byte accesses when possible), L2 only
template <int N>
__device__ __forceinline__ void store_trace(double *dst, const double (&t)[N]) {
  if constexpr (N % 2 == 0) {
#pragma unroll
    for (int j = 0; j < N; j += 2) __stcg(reinterpret_cast<double2 *>(dst + j), make_double2(t[j], t[j + 1]));
  } else {
#pragma unroll
    for (int j = 0; j < N; ++j) __stcg(dst + j, t[j]);
  }
}
template <int N>
__device__ __forceinline__ void load_trace(const double *src, double (&t)[N]) {
  if constexpr (N % 2 == 0) {
#pragma unroll
    for (int j = 0; j < N; j += 2) {
      const double2 v = __ldcg(reinterpret_cast<const double2 *>(src + j));
      t[j] = v.x;
      t[j + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int j = 0; j < N; ++j) t[j] = __ldcg(src + j);
  }
}

// Publish the downwind trace of dim X (ring / far storage); for a ring slot first make sure the
// slot's previous item has been consumed (its consumers, the item itself for dim 0 and the item
// istride_X later, published the following phase).
template <int D, int N, int PH>
__device__ __forceinline__ void publish_trace(const CellParams &p, int X, int b, int k, int r, int C,
                                              const double (&t)[N]) {
  using G = CGeo<D, N>;
  constexpr int NPH1 = G::NPH + 1;
  const int mode = p.tmode[X];
  const int slot = mode == kTraceRing ? (b & p.rmask[X]) : b;
  if (mode == kTraceRing && b > p.rmask[X]) {
    const int old = b - p.rmask[X] - 1;
    wait_flag(p.flags + (size_t)old * NPH1 + PH + 1, p.target);
    wait_flag(p.flags + (size_t)(old + p.istride[X]) * NPH1 + PH + 1, p.target);
  }
  store_trace<N>(p.tbuf[X] + ((size_t)slot * C + k) * G::FN + (size_t)N * r, t);
}

// Non-blocking attempt to read the published upwind trace of dim X (true if it was available).
template <int D, int N, int PH>
__device__ __forceinline__ bool try_trace(const CellParams &p, const CellInfo &ci, int X, int r, int C,
                                          double (&t)[N]) {
  using G = CGeo<D, N>;
  constexpr int NPH1 = G::NPH + 1;
  const int pi = ci.pitem[X];
  if (ld_acquire(p.flags + (size_t)pi * NPH1 + PH) < p.target) return false;
  const int slot = p.tmode[X] == kTraceRing ? (pi & p.rmask[X]) : pi;
  load_trace<N>(p.tbuf[X] + ((size_t)slot * C + ci.pk[X]) * G::FN + (size_t)N * r, t);
  return true;
}

// Upwind trace of dim X for this thread's lines: from the producer (blocking), or directly from the
// neighbour cell (lines along X with stride SX, indexed by the partner digit with stride SY).
template <int D, int N, int PH, int SX, int SY>
__device__ __forceinline__ void upwind_trace(const CellParams &p, const CellInfo &ci, int X, int sg, int R, int r,
                                             int C, double (&t)[N]) {
  using G = CGeo<D, N>;
  constexpr int NPH1 = G::NPH + 1;
  if (ci.direct[X]) {
    const double *nb = p.u + (size_t)ci.nbcell[X] * G::ND + R;
    const double *tau = c_tab[N].tau[sg];
#pragma unroll
    for (int l = 0; l < N; ++l) {
      double s = tau[0] * __ldg(nb + l * SY);
#pragma unroll
      for (int j = 1; j < N; ++j) s = fma(tau[j], __ldg(nb + j * SX + l * SY), s);
      t[l] = s;
    }
  } else {
    const int pi = ci.pitem[X];
    wait_flag(p.flags + (size_t)pi * NPH1 + PH, p.target);
    const int slot = p.tmode[X] == kTraceRing ? (pi & p.rmask[X]) : pi;
    load_trace<N>(p.tbuf[X] + ((size_t)slot * C + ci.pk[X]) * G::FN + (size_t)N * r, t);
  }
}

// One pass over the tile lines of dim P (lines along the first tile index a, one per partner
// digit b): each line is read from smem once and yields both the downwind trace t[b] and the
// volume contribution acc[a][b] (+)= s[b] sum_j K[a][j] u[j][b].
template <int N, int S, bool INIT, class Get>
__device__ __forceinline__ void pass_P(double (&acc)[N][N], Get get, double s0, double sl, double (&t)[N]) {
  const Tables1D &T = c_tab[N];
#pragma unroll
  for (int b = 0; b < N; ++b) {
    const double sb = fma(sl, T.xi[b], s0);  // line speed a_P / h_P * dtfac
    double col[N];
#pragma unroll
    for (int j = 0; j < N; ++j) col[j] = get(j, b);
    double tr = T.tau[S][0] * col[0];
#pragma unroll
    for (int j = 1; j < N; ++j) tr = fma(T.tau[S][j], col[j], tr);
    t[b] = tr;
#pragma unroll
    for (int a = 0; a < N; ++a) {
      double y = T.K[S][a][0] * col[0];
#pragma unroll
      for (int j = 1; j < N; ++j) y = fma(T.K[S][a][j], col[j], y);
      if constexpr (INIT) acc[a][b] = sb * y;
      else acc[a][b] = fma(sb, y, acc[a][b]);
    }
  }
}
// Same for dim Q (lines along b, one per a).
template <int N, int S, class Get>
__device__ __forceinline__ void pass_Q(double (&acc)[N][N], Get get, double s0, double sl, double (&t)[N]) {
  const Tables1D &T = c_tab[N];
#pragma unroll
  for (int a = 0; a < N; ++a) {
    const double sa = fma(sl, T.xi[a], s0);  // line speed a_Q / h_Q * dtfac
    double row[N];
#pragma unroll
    for (int j = 0; j < N; ++j) row[j] = get(a, j);
    double tr = T.tau[S][0] * row[0];
#pragma unroll
    for (int j = 1; j < N; ++j) tr = fma(T.tau[S][j], row[j], tr);
    t[a] = tr;
#pragma unroll
    for (int b = 0; b < N; ++b) {
      double y = T.K[S][b][0] * row[0];
#pragma unroll
      for (int j = 1; j < N; ++j) y = fma(T.K[S][b][j], row[j], y);
      acc[a][b] = fma(sa, y, acc[a][b]);
    }
  }
}

template <int D, int N, int MODE, int PH>
__device__ __forceinline__ void run_phase(const CellParams &p, const CellInfo &ci, const double *stab, int b,
                                          int k, int r, int C, const double *U, double *ACC, bool warp_leader,
                                          bool active) {
  using G = CGeo<D, N>;
  constexpr int P = G::P(PH), Q = G::Q(PH);
  constexpr bool QA = G::QA(PH);
  constexpr int SP = ipow(N, P), SQ = ipow(N, Q);
  constexpr bool FIRST = PH == 0, LAST = PH == G::NPH - 1;
  constexpr int NPH1 = G::NPH + 1;
  // compile-time property: the tile base is a multiple of 16 (all rest strides and n^d are)
  constexpr bool EB16 = (G::ND % 16 == 0) && [] {
    bool ok = true;
    for (int j = 0; j < D; ++j)
      if (j != P && j != Q && ipow(N, j) % 16 != 0) ok = false;
    return ok;
  }();
  const Tables1D &T = c_tab[N];

  ThreadPhase tp;
  thread_phase<D, N, PH, LAST && MODE == kModeAdvection>(p, r, stab, stab + 8, tp);
  const int R = tp.R;
  const int eb = k * G::ND + R;
  const int peb = padded(eb);
  const int sgP = ci.sg[P], sgQ = ci.sg[Q];
  const size_t g0 = (size_t)ci.cell * G::ND + R;
  double acc[N][N];
  double tP[N], tQ[N];
  bool haveP = false, haveQ = false;
  // line speeds (a_i / h_i) * dtfac = s0 + sl * xi_line: a_i varies only with the coordinates of
  // the other dims
  const double facP = p.dtfac * p.inv_h[P], facQ = p.dtfac * p.inv_h[Q];
  const double s0P = (ci.base[P] + tp.wP) * facP, slP = p.a_lin[P][Q] * p.h[Q] * facP;
  const double s0Q = (ci.base[Q] + tp.wQ) * facQ, slQ = p.a_lin[Q][P] * p.h[P] * facQ;
  const bool dirP = ci.direct[P], dirQ = ci.direct[Q];
  if (active) {
    // early attempt at the upwind traces: producers istride items back are usually done, and the
    // loads then overlap the passes below
#if HD_EARLY_TRACES
    if (!dirP && ci.pitem[P] != b) haveP = try_trace<D, N, PH>(p, ci, P, r, C, tP);
    if constexpr (QA) {
      if (!dirQ && ci.pitem[Q] != b) haveQ = try_trace<D, N, PH>(p, ci, Q, r, C, tQ);
    }
#endif
    if constexpr (!FIRST) load_tile<N, SP, SQ, EB16>(ACC, eb, acc);
    // 1./2. volume terms of P and Q and this cell's downwind traces along P and Q -> publish
    double trP[N], trQ[N];
    if constexpr (P == 0 && Q == 1 && EB16 && N * N <= 16 && N % 2 == 0) {
      // contiguous tile (dims 0 and 1): 16-byte loads into registers, conflict-free in the padding
      double uv[N][N];
#pragma unroll
      for (int e = 0; e < N * N; e += 2) {
        const double2 v = *reinterpret_cast<const double2 *>(U + peb + e);
        uv[e % N][e / N] = v.x;
        uv[(e + 1) % N][(e + 1) / N] = v.y;
      }
      auto get = [&](int a, int bb) { return uv[a][bb]; };
      if (sgP == 0) pass_P<N, 0, FIRST>(acc, get, s0P, slP, trP);
      else pass_P<N, 1, FIRST>(acc, get, s0P, slP, trP);
      if constexpr (QA) {
        if (sgQ == 0) pass_Q<N, 0>(acc, get, s0Q, slQ, trQ);
        else pass_Q<N, 1>(acc, get, s0Q, slQ, trQ);
      }
    } else {
      auto get = [&](int a, int bb) { return U[paddr<EB16>(a * SP + bb * SQ, eb, peb)]; };
      if (sgP == 0) pass_P<N, 0, FIRST>(acc, get, s0P, slP, trP);
      else pass_P<N, 1, FIRST>(acc, get, s0P, slP, trP);
      if constexpr (QA) {
        if (sgQ == 0) pass_Q<N, 0>(acc, get, s0Q, slQ, trQ);
        else pass_Q<N, 1>(acc, get, s0Q, slQ, trQ);
      }
    }
    if (p.tmode[P] != kTraceNone) publish_trace<D, N, PH>(p, P, b, k, r, C, trP);
    if constexpr (QA) {
      if (p.tmode[Q] != kTraceNone) publish_trace<D, N, PH>(p, Q, b, k, r, C, trQ);
    }
    if constexpr (LAST && MODE == kModeRK && !HD_DU_DIRECT) {
      // dU of the tile -> this thread's own ACC positions (already consumed), asynchronously; read
      // back in the epilogue, so its HBM latency overlaps the upwind-trace work
#pragma unroll
      for (int a = 0; a < N; ++a)
#pragma unroll
        for (int bb = 0; bb < N; ++bb)
          cp_async8(ACC + paddr<EB16>(a * SP + bb * SQ, eb, peb), p.du + g0 + a * SP + bb * SQ);
      cp_async_commit();
    }
  }
  // publish: one release per warp and phase (only phases somebody waits for)
  if ((p.pubmask >> PH) & 1) {
    __syncwarp();
    if (warp_leader) red_release_add(p.flags + (size_t)b * NPH1 + PH);
  }
  if (!active) return;

  // 3./4. upwind traces and rank-1 lifts
  if (!haveP) upwind_trace<D, N, PH, SP, SQ>(p, ci, P, sgP, R, r, C, tP);
#pragma unroll
  for (int bb = 0; bb < N; ++bb) tP[bb] *= fma(slP, T.xi[bb], s0P);
  if (sgP == 0) lift_P<N, 0>(acc, tP);
  else lift_P<N, 1>(acc, tP);
  if constexpr (QA) {
    if (!haveQ) upwind_trace<D, N, PH, SQ, SP>(p, ci, Q, sgQ, R, r, C, tQ);
#pragma unroll
    for (int a = 0; a < N; ++a) tQ[a] *= fma(slQ, T.xi[a], s0Q);
    if (sgQ == 0) lift_Q<N, 0>(acc, tQ);
    else lift_Q<N, 1>(acc, tQ);
  }

  if constexpr (!LAST) {
#pragma unroll
    for (int a = 0; a < N; ++a)
#pragma unroll
      for (int bb = 0; bb < N; ++bb) ACC[paddr<EB16>(a * SP + bb * SQ, eb, peb)] = acc[a][bb];
  } else if constexpr (MODE == kModeAdvection) {
    // weak form: v = M (M^-1 A u), M_qq = |J| prod_i w_{q_i}
    const double wr = tp.wr;
#pragma unroll
    for (int a = 0; a < N; ++a)
#pragma unroll
      for (int bb = 0; bb < N; ++bb) __stcs(p.out + g0 + a * SP + bb * SQ, acc[a][bb] * (wr * (T.w[a] * T.w[bb])));
  } else {
    // LSRK 2N stage: dU <- A_s dU + dt M^-1 A(U); U_new <- U + B_s dU
    if constexpr (MODE == kModeRK && !HD_DU_DIRECT) cp_async_wait<0>();
#pragma unroll
    for (int a = 0; a < N; ++a)
#pragma unroll
      for (int bb = 0; bb < N; ++bb) {
        const int o = paddr<EB16>(a * SP + bb * SQ, eb, peb);
        double dun = acc[a][bb];
        if constexpr (MODE == kModeRK)
          dun = fma(p.rk_a, HD_DU_DIRECT ? __ldcs(p.du + g0 + a * SP + bb * SQ) : ACC[o], dun);
        __stcs(p.du + g0 + a * SP + bb * SQ, dun);
        __stcs(p.out + g0 + a * SP + bb * SQ, fma(p.rk_b, dun, U[o]));
      }
  }
}

// One item (all phases). Not inlined into the persistent loop, so that item-invariant values are
// not hoisted out of it and kept live in registers across the whole loop.
template <int D, int N, int MODE>
__device__ __noinline__ void process_item(const CellParams &p, const CellInfo &ci, const double *stab, int b,
                                          int k, int r, int C, const double *U, double *ACC, bool warp_leader,
                                          bool active) {
  using G = CGeo<D, N>;
  run_phase<D, N, MODE, 0>(p, ci, stab, b, k, r, C, U, ACC, warp_leader, active);
  if constexpr (G::NPH > 1) {
    __syncthreads();
    run_phase<D, N, MODE, (G::NPH > 1 ? 1 : 0)>(p, ci, stab, b, k, r, C, U, ACC, warp_leader, active);
  }
  if constexpr (G::NPH > 2) {
    __syncthreads();
    run_phase<D, N, MODE, (G::NPH > 2 ? 2 : 0)>(p, ci, stab, b, k, r, C, U, ACC, warp_leader, active);
  }
}

template <int D, int N, int MODE>
__global__ void __launch_bounds__(256, 2) cell_kernel(const __grid_constant__ CellParams p, int C) {
  using G = CGeo<D, N>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const int bufp = padded(((C * G::ND + 15) / 16) * 16);
  double *smem = reinterpret_cast<double *>(smem_raw);
  double *ACC = smem + 2 * bufp;
  double *stab = ACC + bufp;                                        // xi[8], w[8]
  CellInfo *info = reinterpret_cast<CellInfo *>(stab + 16);         // C entries
  const int tid = threadIdx.x;
  const int k = tid / G::NT;
  const int r = tid - k * G::NT;
  const bool active = k < C;
  const int lane = tid & 31;
  const bool warp_leader = lane == 0 && (tid - lane) < C * G::NT;
  if (tid < 8) {
    stab[tid] = tid < N ? c_tab[N].xi[tid] : 0.0;
    stab[8 + tid] = tid < N ? c_tab[N].w[tid] : 0.0;
  }

  int b = blockIdx.x;
  if (b >= p.nitems) return;
  auto copy_item = [&](int first_cell, double *dst) {
    const double *src = p.u + (size_t)first_cell * G::ND;
    const int total = C * G::ND;
    if constexpr (G::ND % 2 == 0) {
      for (int i = tid; i < (total >> 1); i += blockDim.x) cp_async16(dst + padded(2 * i), src + 2 * i);
    } else {
      for (int i = tid; i < total; i += blockDim.x) cp_async8(dst + padded(i), src + i);
    }
  };
  copy_item(item_first_cell<D>(p, b, C), smem);
  cp_async_commit();
  for (int it = 0; b < p.nitems; b += gridDim.x, ++it) {
    const int bn = b + gridDim.x;
    __syncthreads();  // previous item finished: info and the other U buffer are free
    if (bn < p.nitems) copy_item(item_first_cell<D>(p, bn, C), smem + ((it + 1) & 1) * bufp);
    cp_async_commit();
    decode_coords<D>(p, b, C, info);
    __syncthreads();
    decode_links<D>(p, b, C, info);
    cp_async_wait<1>();
    __syncthreads();
    const double *U = smem + (it & 1) * bufp;
    process_item<D, N, MODE>(p, info[active ? k : 0], stab, b, k, r, C, U, ACC, warp_leader, active);
    // item done: publish phase NPH (ring slots of the last phase use it as "finished reading")
    if ((p.pubmask >> G::NPH) & 1) {
      __syncwarp();
      if (warp_leader) red_release_add(p.flags + (size_t)b * (G::NPH + 1) + G::NPH);
    }
  }
  cp_async_wait<0>();
}

}  // namespace hd
