// hd_cell.cuh -- the fused cell kernel (element-centric loop, Alg. 1/Alg. 2) for sm_100a.
// Included by hd_kernels.cu (single translation unit with the __constant__ tables).
//
// Merged operator: M^-1 A = sum_i (a_i(z)/h_i) L_i along dim i; L_i = the n x n matrix K
// (volume term + own-face upwind term, rows divided by w_m) plus the rank-1 lift lam * (tau . u_nb) of
// the UPWIND neighbour's trace. One CTA iteration processes a GROUP of CT cells that are consecutive
// along dim 0; threads own, per phase, an n x n register tile of a cell over a pair of dims (P, Q).
//
// Work units and upwind traces (the part that decides performance; DESIGN.md §6 "Upwind traces"):
//   * pencil mode (CT | L_1, a_0 independent of z_1): a group is CT cells at one c_0 from CT adjacent
//     pencils, a unit is those pencils, processed group by group by ONE CTA upwind -> downwind (a_0
//     has one sign on the unit). The dim-0 trace of a cell is the previous group's downwind trace,
//     carried in smem.
//   * every other dim whose traversal follows the sign of its speed PUBLISHES its downwind traces
//     (n^(d-1) values, 1/n of a cell) into a per-dim buffer and a per-unit progress flag. Units are
//     swept in direction-following order with a skewed start (pencil_decode), so a unit's upwind
//     neighbours in the same round run `skew` groups ahead: when a group starts, the traces it needs
//     were written a few groups earlier and are usually still in L2 (optionally discarded after use,
//     HD_DISCARD). A trace that is not published yet (first groups, skew seams, round seams, wraps)
//     is formed from the neighbour cell itself (direct read). Nobody ever waits for another CTA.
//   * multi-pencil mode (L_0 | CT, small d): a group holds whole pencils; in-group neighbours come
//     from smem, the rest by direct reads. Chunk mode (CT | L_0, when a_0 depends on z_1 and a pencil
//     does not fit one group) is the same with part of a pencil per group.
#pragma once
#ifndef HD_MINB
#define HD_MINB 1
#endif

namespace hd {

enum TraceSrc : unsigned char { kSrcDirect = 0, kSrcGroup = 1, kSrcCarry = 2, kSrcPub = 3, kSrcHalo = 4 };
enum TraceOut : unsigned char { kOutNone = 0, kOutCarry = 1, kOutPub = 2 };

// Shared-memory layout of a cell: element (d_0, ..., d_{D-1}) at sum_i d_i S_i -- ADDITIVE, so a thread's
// tile element is its rest offset plus a compile-time constant (base + immediate addressing, no
// per-element index arithmetic). The padded strides (tools/smem_layout.py; pinned by
// tests/test_smem_layout.py) keep the layout injective (mixed radix), keep 16-byte pairs along dim 0
// aligned (N even: S_i even for i >= 1) and make the tile accesses of every phase as conflict-free as
// the earlier XOR swizzle or better; other (D, N) keep the plain strides N^i.
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
  // one cell must fit the smem pipeline (cell_smem_bytes with CT = 1; cell info etc. < 2 KB): n^d <= 4096
  static constexpr bool OK = NT <= 256 && (3 * NDP + FN + 16 + NPH * 1024) * 8 + 2048 + 1024 <= 227 * 1024;
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

// element T (a compile-time offset whose digits are disjoint from the thread's rest offset R,
// sR = swz(R)) of a cell buffer: the layout is additive, so this folds to sR + constant
template <int D, int N>
__device__ __forceinline__ constexpr int sidx(int sR, int T) {
  return sR + swz<D, N>(T);
}

struct CellInfo {
  double base[kMaxD];        // a_i at the cell's lower corner
  int cell;                  // local memory index of the cell
  int cu;                    // cell slot inside its unit (trace-buffer addressing)
  int unit;                  // the unit being processed (kOutPub slot)
  int nb[kMaxD];             // kSrcDirect: neighbour cell index; kSrcGroup: neighbour slot k' in the group
  int slot[kMaxD];           // kSrcPub: producer trace index (unit * UC + cell slot); kSrcHalo: receive slot
  const double *tsrc[kMaxD]; // kSrcPub / kSrcHalo: the trace to read (else null)
  int pflag[kMaxD];          // pending publication check: producer unit (-1: none)
  int need[kMaxD];           // ... and the flag value that means "the neighbour's step is done"
  unsigned char src[kMaxD];  // TraceSrc of the upwind trace per dim
  unsigned char out[kMaxD];  // TraceOut of the downwind trace per dim
  unsigned char sg[kMaxD];   // 1: a_i < 0 on this cell (upwind neighbour at +e_i)
  unsigned char pad[2];
};

// Pencil-mode decode of one unit, cached in smem for all its groups (pencil_decode, plus for each
// published dim the producer unit of the upwind neighbours and its direction / start).
struct UnitInfo {
  int c[kMaxD], t[kMaxD];
  int base, dir0, skew;
  int pu[kMaxD], pdir0[kMaxD], pskew[kMaxD];
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
// Bring a whole neighbour cell (contiguous, 16-byte multiple) into L2 ahead of a direct read.
__device__ __forceinline__ void prefetch_l2(const void *p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ void discard_l2_line(const void *p) {
  asm volatile("discard.global.L2 [%0], 128;\n" ::"l"(p) : "memory");
}

// sign of a_i on a cell with coordinates c (local box; global = c + coff), evaluated at the cell centre
// (constant on the cell by reading C11). The host plan (hd_plan.cpp) evaluates the same fma sequence.
template <int D>
__device__ __forceinline__ void cell_speed(const CellParams &p, int i, const int (&c)[kMaxD], double &base, int &sg) {
  double ab = p.a_const[i], half = 0.0;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    ab = fma(p.a_lin[i][j], fma((double)(c[j] + p.coff[j]), p.h[j], p.lo[j]), ab);
    half = fma(p.a_lin[i][j], 0.5 * p.h[j], half);
  }
  base = ab;
  sg = (ab + half) < 0.0 ? 1 : 0;
}

// Pencil mode: a group is CT cells at the same c_0 from CT adjacent pencils (along dim 1); a unit is those
// CT pencils, processed one c_0 position (group) per step.
// Pencil-mode unit decode, slowest dim first: traversal coordinates t_j = (u / ustride_j) % L_j; a dim
// that "follows" its speed (the sign of a_j depends only on slower dims, so it is constant along the
// sweep) is traversed upwind -> downwind: c_j = L_j - 1 - t_j where a_j < 0. Then every upwind neighbour
// along such a dim is an EARLIER unit. Returns the pencil's base cell, the dim-0 direction (1: a_0 < 0,
// groups from the far end) and the start: the pencil starts at group (-K sum_j t_j) mod GPU (K = p.skew),
// so a unit's upwind neighbours along every dim (same round) run K groups ahead of it.
template <int D>
__device__ __forceinline__ int pencil_decode(const CellParams &p, int u, int (&c)[kMaxD], int (&t)[kMaxD], int &dir0,
                                             int &skew) {
  int base = 0, tsum = 0;
#pragma unroll
  for (int j = 0; j < kMaxD; ++j) {
    c[j] = 0;
    t[j] = 0;
  }
#pragma unroll
  for (int j = D - 1; j >= 1; --j) {
    // dim 1 is traversed in blocks of CT cells (the cells of one group)
    const int ext = j == 1 ? p.L[1] / p.CT : p.L[j];
    const int tj = (u / p.ustride[j]) % ext;
    t[j] = tj;
    tsum += tj;
    int neg = 0;
    if (p.follow[j]) {
      double b;
      cell_speed<D>(p, j, c, b, neg);  // faster coordinates are still 0: a_j does not depend on them
    }
    const int cj = neg ? ext - 1 - tj : tj;
    c[j] = j == 1 ? cj * p.CT : cj;
    base += c[j] * p.lstride[j];
  }
  double b0;
  cell_speed<D>(p, 0, c, b0, dir0);
  skew = (p.GPU - (p.skew * tsum) % p.GPU) % p.GPU;
  return base;
}

// Unit index (pencil mode) of the unit holding a cell with coordinates c.
template <int D>
__device__ __forceinline__ int unit_of(const CellParams &p, const int (&c)[kMaxD]) {
  int cc[kMaxD], u = 0;
#pragma unroll
  for (int j = 0; j < kMaxD; ++j) cc[j] = 0;
#pragma unroll
  for (int j = D - 1; j >= 1; --j) {
    int neg = 0;
    if (p.follow[j]) {
      double b;
      cell_speed<D>(p, j, cc, b, neg);
    }
    cc[j] = c[j];
    const int ext = j == 1 ? p.L[1] / p.CT : p.L[j];
    const int cj = j == 1 ? c[1] / p.CT : c[j];
    u += (neg ? ext - 1 - cj : cj) * p.ustride[j];
  }
  return u;
}

// memory group of processing step gi of a unit with direction dir0 and skew
__device__ __forceinline__ int step_group(const CellParams &p, int gi, int dir0, int skew) {
  const int g = (gi + skew) % p.GPU;
  return dir0 ? p.GPU - 1 - g : g;
}
// processing step of memory group g
__device__ __forceinline__ int group_step(const CellParams &p, int g, int dir0, int skew) {
  const int gg = dir0 ? p.GPU - 1 - g : g;
  return (gg - skew + p.GPU) % p.GPU;
}

// Unit decode for the cache: thread j computes the unit (redundantly) and, for a published dim j, its
// producer unit; thread 0 writes the unit fields.
template <int D>
__device__ __forceinline__ void decode_unit(const CellParams &p, int u, int j, UnitInfo &ui) {
  int c[kMaxD], t[kMaxD], dir0, skew;
  const int base = pencil_decode<D>(p, u, c, t, dir0, skew);
  if (j == 0) {
#pragma unroll
    for (int q = 0; q < kMaxD; ++q) {
      ui.c[q] = c[q];
      ui.t[q] = t[q];
    }
    ui.base = base;
    ui.dir0 = dir0;
    ui.skew = skew;
  }
  if (j >= 1 && j < D && p.pub[j]) {
    // the upwind neighbour along j of every cell of this pencil sits in one pencil (a_j does not
    // depend on z_0 or z_j): its unit, direction and start
    double b;
    int sg;
    cell_speed<D>(p, j, c, b, sg);
    int cn[kMaxD];
#pragma unroll
    for (int q = 0; q < kMaxD; ++q) cn[q] = c[q];
    // the unit's boundary cell along dim 1 (its upwind end) reaches into the neighbouring block
    if (j == 1) cn[1] = sg ? c[1] + p.CT - 1 : c[1];
    cn[j] = cn[j] + (sg ? 1 : -1);
    int pu = -1, pd = 0, ps = 0;
    if (cn[j] >= 0 && cn[j] < p.L[j]) {
      pu = unit_of<D>(p, cn);
      int pc[kMaxD], pt[kMaxD];
      pencil_decode<D>(p, pu, pc, pt, pd, ps);
      if (pu >= u) pu = -1;  // not an earlier unit (a dim that does not follow): never published in time
    }
    ui.pu[j] = pu;
    ui.pdir0[j] = pd;
    ui.pskew[j] = ps;
  }
}

// Decode dim `i` of cell k of group gi of unit u (dim 0 also writes the cell-level fields).
template <int D>
__device__ __forceinline__ void decode_cell(const CellParams &p, const UnitInfo &ui, int u, int gi, int k, CellInfo &ci,
                                            int i) {
  int c[kMaxD];
  int first;
  if (p.pencil) {
#pragma unroll
    for (int j = 0; j < kMaxD; ++j) c[j] = ui.c[j];
    const int g = step_group(p, gi, ui.dir0, ui.skew);
    c[0] = g;
    c[1] += k;
    first = ui.base + g;
  } else {
    first = u * p.CT;
    int rr = first + k;
#pragma unroll
    for (int j = 0; j < kMaxD; ++j) c[j] = 0;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      c[j] = rr % p.L[j];
      rr /= p.L[j];
    }
  }
  int cell = 0;
#pragma unroll
  for (int j = 0; j < D; ++j) cell += c[j] * p.lstride[j];
  if (i == 0) {
    ci.cell = cell;
    ci.unit = u;
    ci.cu = p.pencil ? k * p.L[0] + c[0] : k;
  }
  double base;
  int sg;
  cell_speed<D>(p, i, c, base, sg);
  ci.base[i] = base;
  ci.sg[i] = (unsigned char)sg;
  const int up = sg ? 1 : -1;
  int cn = c[i] + up;
  const bool outside = cn < 0 || cn >= p.L[i];
  if (cn < 0) cn += p.L[i];
  if (cn >= p.L[i]) cn -= p.L[i];
  const int nbcell = cell + (cn - c[i]) * p.lstride[i];
  unsigned char src = kSrcDirect, out = kOutNone;
  int nb = nbcell, slot = 0, pflag = -1, need = 0;
  if (i == 0 && p.pencil) {
    // every cell of a group feeds the carry of its pencil's next step
    if (gi < p.GPU - 1) out = kOutCarry;
  }
  if (i > 0 && p.pub[i]) {
    // downwind neighbour inside the local box and outside this group: publish (its consumer runs a
    // few steps later)
    const int cd = c[i] - up;
    const bool in_group = p.pencil && i == 1 && k - up >= 0 && k - up < p.CT;
    if (cd >= 0 && cd < p.L[i] && !in_group) out = kOutPub;
  }
  if (outside && p.xsplit[i]) {
    // the upwind neighbour lives on another rank: its trace arrived in the halo buffer
    src = kSrcHalo;
    const int ls = p.lstride[i];
    slot = p.hslot[i][(cell % ls) + (cell / (ls * p.L[i])) * ls];
  } else if (i == 0 && p.pencil) {
    if (gi > 0) src = kSrcCarry;  // the previous step processed the upwind neighbour along dim 0
  } else if (p.pencil && i == 1 && k + up >= 0 && k + up < p.CT) {
    src = kSrcGroup;  // the neighbour pencil is in this group
    nb = k + up;
  } else if (!p.pencil && nbcell >= first && nbcell < first + p.CT) {
    src = kSrcGroup;
    nb = nbcell - first;
  } else if (p.pub[i] && !outside && ui.pu[i] >= 0) {
    // the producer finished the step that processed the neighbour's group (the flag counts the steps
    // completed in this launch)?
    // publication check left pending (resolve_cell): the producer unit, the flag value meaning "the
    // step that processed the neighbour's group is done", and the neighbour's slot in the producer
    // unit (same pencil and c_0, except along dim 1 where it is the other end of the neighbouring block)
    pflag = ui.pu[i];
    need = p.epoch | (group_step(p, c[0], ui.pdir0[i], ui.pskew[i]) + 1);
    const int kn = (p.pencil && i == 1) ? (k + up + p.CT) % p.CT : k;
    slot = pflag * p.UC + (p.pencil ? kn * p.L[0] + c[0] : kn);
  }
  if (src == kSrcDirect && pflag < 0 && p.prefetch)
    prefetch_l2(p.u + (size_t)nb * p.ND, (unsigned)(p.ND * 8));
  ci.src[i] = src;
  ci.out[i] = out;
  ci.nb[i] = nb;
  ci.slot[i] = slot;
  ci.pflag[i] = pflag;
  ci.need[i] = need;
  ci.tsrc[i] = src == kSrcHalo ? p.hbuf[i] + (size_t)slot * p.FN : nullptr;
}

// Resolve a pending publication check with the producer's flag value fv (fetched asynchronously).
// Flags only grow within a launch (and a flag of an older launch is smaller), so a stale value can only
// make the check fail, which falls back to a direct read.
__device__ __forceinline__ void resolve_cell(const CellParams &p, CellInfo &ci, int i, int fv) {
  if (ci.pflag[i] >= 0 && fv >= ci.need[i]) {
    ci.src[i] = kSrcPub;
    ci.tsrc[i] = p.tbuf[i] + (size_t)ci.slot[i] * p.FN;
  } else if (ci.pflag[i] >= 0 && p.prefetch) {
    prefetch_l2(p.u + (size_t)ci.nb[i] * p.ND, (unsigned)(p.ND * 8));  // will be read directly
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
      wP = fma(p.a_lin[P][j] * p.h[j], sx[m], wP);
      wQ = fma(p.a_lin[Q][j] * p.h[j], sx[m], wQ);
      if constexpr (MASS) wr *= sw[m];
    }
    nj *= N;
  }
  tp.wP = wP;
  tp.wQ = wQ;
  tp.wr = wr;
  tp.R = R;
}

// One pass over the tile lines of dim P (lines along the first tile index a, one per partner digit
// b): yields the downwind trace t[b] = tau . line and the volume contribution
// acc[a][b] (+)= s_b sum_j K[a][j] u[j][b].
template <int N, int S, bool INIT, bool TRACE>
__device__ __forceinline__ void pass_P(double (&acc)[N][N], const double (&uv)[N][N], double s0, double sl,
                                       double (&t)[N]) {
  const Tables1D &T = c_tab[N];
#pragma unroll
  for (int b = 0; b < N; ++b) {
    const double sb = fma(sl, T.xi[b], s0);
    if constexpr (TRACE) {
      double tr = T.tau[S][0] * uv[0][b];
#pragma unroll
      for (int j = 1; j < N; ++j) tr = fma(T.tau[S][j], uv[j][b], tr);
      t[b] = tr;
    }
    // j outer, a inner: N independent accumulation chains per step (latency-friendly order)
    double y[N];
#pragma unroll
    for (int a = 0; a < N; ++a) y[a] = T.K[S][a][0] * uv[0][b];
#pragma unroll
    for (int j = 1; j < N; ++j)
#pragma unroll
      for (int a = 0; a < N; ++a) y[a] = fma(T.K[S][a][j], uv[j][b], y[a]);
#pragma unroll
    for (int a = 0; a < N; ++a) {
      if constexpr (INIT) acc[a][b] = sb * y[a];
      else acc[a][b] = fma(sb, y[a], acc[a][b]);
    }
  }
}
// Same for dim Q (lines along b, one per a).
template <int N, int S, bool TRACE>
__device__ __forceinline__ void pass_Q(double (&acc)[N][N], const double (&uv)[N][N], double s0, double sl,
                                       double (&t)[N]) {
  const Tables1D &T = c_tab[N];
#pragma unroll
  for (int a = 0; a < N; ++a) {
    const double sa = fma(sl, T.xi[a], s0);
    if constexpr (TRACE) {
      double tr = T.tau[S][0] * uv[a][0];
#pragma unroll
      for (int j = 1; j < N; ++j) tr = fma(T.tau[S][j], uv[a][j], tr);
      t[a] = tr;
    }
    double y[N];
#pragma unroll
    for (int b = 0; b < N; ++b) y[b] = T.K[S][b][0] * uv[a][0];
#pragma unroll
    for (int j = 1; j < N; ++j)
#pragma unroll
      for (int b = 0; b < N; ++b) y[b] = fma(T.K[S][b][j], uv[a][j], y[b]);
#pragma unroll
    for (int b = 0; b < N; ++b) acc[a][b] = fma(sa, y[b], acc[a][b]);
  }
}

// Upwind trace of this thread's N face points along dim X (stride SX), the face points being indexed by
// the partner tile digit l (stride SY): t[l] = sum_j tau[j] u_nb[R + j SX + l SY]. Same summation order
// as the producer's pass, so every source yields the same bits.
template <int D, int N, int SX, int SY>
__device__ __forceinline__ void trace_global(const double *nb, int S, double (&t)[N]) {
  const double *tau = c_tab[N].tau[S];
  double v[N][N];
#pragma unroll
  for (int l = 0; l < N; ++l)
#pragma unroll
    for (int j = 0; j < N; ++j) v[l][j] = __ldg(nb + j * SX + l * SY);
#pragma unroll
  for (int l = 0; l < N; ++l) {
    double s = tau[0] * v[l][0];
#pragma unroll
    for (int j = 1; j < N; ++j) s = fma(tau[j], v[l][j], s);
    t[l] = s;
  }
}
template <int D, int N, int SX, int SY>
__device__ __forceinline__ void trace_smem(const double *cellbuf, int sR, int S, double (&t)[N]) {
  const double *tau = c_tab[N].tau[S];
#pragma unroll
  for (int l = 0; l < N; ++l) {
    double s = tau[0] * cellbuf[sidx<D, N>(sR, l * SY)];
#pragma unroll
    for (int j = 1; j < N; ++j) s = fma(tau[j], cellbuf[sidx<D, N>(sR, j * SX + l * SY)], s);
    t[l] = s;
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

// Early part of the upwind trace of dim X: the sources that are a plain N-value load -- the carry (smem)
// and the published / halo traces (global, L2: issued before the passes so the latency hides behind
// them). In-group (smem) and direct (global) traces are contracted after the passes.
template <int D, int N>
__device__ __forceinline__ void trace_early(const CellInfo &ci, int X, int r, const double *carry_in, double (&t)[N]) {
  switch (ci.src[X]) {
    case kSrcCarry:
      load_vec<N>(carry_in + N * r, t, false);
      break;
    case kSrcPub:
    case kSrcHalo:
      load_vec<N>(ci.tsrc[X] + N * r, t, true);
      break;
    default:
      break;
  }
}

// Smem pointers of one group: its cells (U), the running accumulator and the dim-0 carry.
struct GroupBufs {
  const double *U;
  double *ACC;
  const double *carry_in;
  double *carry_out;
};

// The per-thread constants of every phase (thread_phase, plus the swizzled rest offset), once per
// launch into this thread's column of the smem table read by run_phase.
template <int D, int N, int MODE, int PH>
__device__ __forceinline__ void phase_entry(const CellParams &p, int r, double *ptab) {
  using G = CGeo<D, N>;
  ThreadPhase tp;
  thread_phase<D, N, PH, PH == G::NPH - 1 && MODE == kModeAdvection>(p, r, c_tab[N].xi, c_tab[N].w, tp);
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

template <int D, int N, int MODE, int PH>
__device__ __forceinline__ void run_phase(const CellParams &p, const CellInfo &ci, const double *ptab, int k, int r,
                                          const GroupBufs &gb, bool active) {
  if (!active) return;  // padding threads of the CTA: only the barriers between phases
  using G = CGeo<D, N>;
  constexpr int P = G::P(PH), Q = G::Q(PH);
  constexpr bool QA = G::QA(PH);
  constexpr int SP = ipow(N, P), SQ = ipow(N, Q);
  constexpr bool FIRST = PH == 0, LAST = PH == G::NPH - 1;
  const Tables1D &T = c_tab[N];

  // per-thread phase constants, computed once per launch (phase_table): [PH][wP | wQ | wr | (R, sR)][256]
  ThreadPhase tp;
  const int tid = (int)threadIdx.x;
  const double *pt = ptab + PH * 1024;
  tp.wP = pt[tid];
  tp.wQ = pt[256 + tid];
  tp.wr = pt[512 + tid];
  const int2 rs = reinterpret_cast<const int2 *>(pt + 768)[tid];
  const int R = rs.x;
  const int sR = rs.y;
  const double *U = gb.U + (size_t)k * G::NDP;
  double *A = gb.ACC + (size_t)k * G::NDP;
  const int sgP = ci.sg[P], sgQ = ci.sg[Q];
  const size_t g0 = (size_t)ci.cell * G::ND + R;
  // line speeds (a_i / h_i) * dtfac = s0 + sl * xi_line (a_i varies only with the other dims)
  const double facP = p.dtfac * p.inv_h[P], facQ = p.dtfac * p.inv_h[Q];
  const double s0P = (ci.base[P] + tp.wP) * facP, slP = p.a_lin[P][Q] * p.h[Q] * facP;
  const double s0Q = (ci.base[Q] + tp.wQ) * facQ, slQ = p.a_lin[Q][P] * p.h[P] * facQ;

  // carry / published / halo traces, read before the passes (the carry may then be overwritten in place)
  double tP[N], tQ[N];
  trace_early<D, N>(ci, P, r, gb.carry_in, tP);
  if constexpr (QA) trace_early<D, N>(ci, Q, r, gb.carry_in, tQ);

  double acc[N][N];
  {
    double uv[N][N];
    if constexpr (P == 0 && N % 2 == 0) {
#pragma unroll
      for (int b = 0; b < N; ++b)
#pragma unroll
        for (int a = 0; a < N; a += 2) {
          const double2 v = *reinterpret_cast<const double2 *>(U + sidx<D, N>(sR, a + b * SQ));
          uv[a][b] = v.x;
          uv[a + 1][b] = v.y;
        }
    } else {
#pragma unroll
      for (int a = 0; a < N; ++a)
#pragma unroll
        for (int b = 0; b < N; ++b) uv[a][b] = U[sidx<D, N>(sR, a * SP + b * SQ)];
    }
    if constexpr (!FIRST) {
#pragma unroll
      for (int a = 0; a < N; ++a)
#pragma unroll
        for (int b = 0; b < N; ++b) acc[a][b] = A[sidx<D, N>(sR, a * SP + b * SQ)];
    }
    if constexpr (LAST && MODE == kModeRK) {
      // dU of the tile -> this thread's own ACC positions (already consumed), asynchronously; read back
      // in the epilogue, so its HBM latency overlaps the passes and the lifts
#pragma unroll
      for (int a = 0; a < N; ++a)
#pragma unroll
        for (int b = 0; b < N; ++b) cp_async8(A + sidx<D, N>(sR, a * SP + b * SQ), p.du + g0 + a * SP + b * SQ);
      cp_async_commit();
    }
    // volume terms of P and Q and this cell's downwind traces along P and Q
    double trP[N], trQ[N];
    const unsigned char oP = ci.out[P], oQ = QA ? ci.out[Q] : (unsigned char)kOutNone;
    if (oP != kOutNone) {
      if (sgP == 0) pass_P<N, 0, FIRST, true>(acc, uv, s0P, slP, trP);
      else pass_P<N, 1, FIRST, true>(acc, uv, s0P, slP, trP);
    } else {
      if (sgP == 0) pass_P<N, 0, FIRST, false>(acc, uv, s0P, slP, trP);
      else pass_P<N, 1, FIRST, false>(acc, uv, s0P, slP, trP);
    }
    if constexpr (QA) {
      if (oQ != kOutNone) {
        if (sgQ == 0) pass_Q<N, 0, true>(acc, uv, s0Q, slQ, trQ);
        else pass_Q<N, 1, true>(acc, uv, s0Q, slQ, trQ);
      } else {
        if (sgQ == 0) pass_Q<N, 0, false>(acc, uv, s0Q, slQ, trQ);
        else pass_Q<N, 1, false>(acc, uv, s0Q, slQ, trQ);
      }
    }
    // publish the downwind traces (dim 0 only ever feeds the carry; it is always P of phase 0)
    if (oP == kOutCarry) store_vec<N>(gb.carry_out + N * r, trP, false);
    else if (oP == kOutPub) store_vec<N>(p.tbuf[P] + ((size_t)ci.unit * p.UC + ci.cu) * G::FN + (size_t)N * r, trP, true);
    if constexpr (QA) {
      if (oQ == kOutPub)
        store_vec<N>(p.tbuf[Q] + ((size_t)ci.unit * p.UC + ci.cu) * G::FN + (size_t)N * r, trQ, true);
    }
  }

  // in-group neighbours (smem) and direct reads of the upwind neighbour (traces not published in time)
  if (ci.src[P] == kSrcGroup) trace_smem<D, N, SP, SQ>(gb.U + (size_t)ci.nb[P] * G::NDP, sR, sgP, tP);
  else if (ci.src[P] == kSrcDirect) {
    if (p.dbg & 1) { for (int l = 0; l < N; ++l) tP[l] = 0.0; }  // timing experiment only
    else trace_global<D, N, SP, SQ>(p.u + (size_t)ci.nb[P] * G::ND + R, sgP, tP);
  }
  if constexpr (QA) {
    if (ci.src[Q] == kSrcGroup) trace_smem<D, N, SQ, SP>(gb.U + (size_t)ci.nb[Q] * G::NDP, sR, sgQ, tQ);
    else if (ci.src[Q] == kSrcDirect) {
      if (p.dbg & 1) { for (int l = 0; l < N; ++l) tQ[l] = 0.0; }  // timing experiment only
      else trace_global<D, N, SQ, SP>(p.u + (size_t)ci.nb[Q] * G::ND + R, sgQ, tQ);
    }
  }

  // rank-1 lifts of the upwind traces
  if (sgP == 0) {
#pragma unroll
    for (int b = 0; b < N; ++b) {
      const double tb = tP[b] * fma(slP, T.xi[b], s0P);
#pragma unroll
      for (int a = 0; a < N; ++a) acc[a][b] = fma(T.lam[0][a], tb, acc[a][b]);
    }
  } else {
#pragma unroll
    for (int b = 0; b < N; ++b) {
      const double tb = tP[b] * fma(slP, T.xi[b], s0P);
#pragma unroll
      for (int a = 0; a < N; ++a) acc[a][b] = fma(T.lam[1][a], tb, acc[a][b]);
    }
  }
  if constexpr (QA) {
    if (sgQ == 0) {
#pragma unroll
      for (int a = 0; a < N; ++a) {
        const double ta = tQ[a] * fma(slQ, T.xi[a], s0Q);
#pragma unroll
        for (int b = 0; b < N; ++b) acc[a][b] = fma(T.lam[0][b], ta, acc[a][b]);
      }
    } else {
#pragma unroll
      for (int a = 0; a < N; ++a) {
        const double ta = tQ[a] * fma(slQ, T.xi[a], s0Q);
#pragma unroll
        for (int b = 0; b < N; ++b) acc[a][b] = fma(T.lam[1][b], ta, acc[a][b]);
      }
    }
  }

  // published traces are consumed exactly once: drop their L2 lines without write-back (one lane per
  // 128-byte line, after the lanes sharing it have their values)
  if constexpr ((N * 8) <= 128 && 128 % (N * 8) == 0) {
    constexpr int TPL = 128 / (N * 8);  // threads per line
    if (p.discard && p.pubany) {
      // lanes of this warp that run the phase (padding threads k >= CT returned at the top)
      const int wb = (int)(threadIdx.x & ~31u), nact = p.CT * G::NT - wb;
      __syncwarp(nact >= 32 ? 0xffffffffu : ((1u << nact) - 1u));
      if (r % TPL == 0) {
        if (ci.src[P] == kSrcPub) discard_l2_line(ci.tsrc[P] + N * r);
        if constexpr (QA) {
          if (ci.src[Q] == kSrcPub) discard_l2_line(ci.tsrc[Q] + N * r);
        }
      }
    }
  }

  if constexpr (!LAST && P == 0 && N % 2 == 0) {
#pragma unroll
    for (int b = 0; b < N; ++b)
#pragma unroll
      for (int a = 0; a < N; a += 2)
        *reinterpret_cast<double2 *>(A + sidx<D, N>(sR, a + b * SQ)) = make_double2(acc[a][b], acc[a + 1][b]);
  } else if constexpr (!LAST) {
#pragma unroll
    for (int a = 0; a < N; ++a)
#pragma unroll
      for (int b = 0; b < N; ++b) A[sidx<D, N>(sR, a * SP + b * SQ)] = acc[a][b];
  } else if constexpr (MODE == kModeAdvection) {
    // weak form: v = M (M^-1 A u), M_qq = |J| prod_i w_{q_i}
    const double wr = tp.wr;
#pragma unroll
    for (int a = 0; a < N; ++a)
#pragma unroll
      for (int b = 0; b < N; ++b) __stcs(p.out + g0 + a * SP + b * SQ, acc[a][b] * (wr * (T.w[a] * T.w[b])));
  } else {
    // LSRK 2N stage: dU <- A_s dU + dt M^-1 A(U); U_new <- U + B_s dU
    if constexpr (MODE == kModeRK) cp_async_wait<0>();
#pragma unroll
    for (int a = 0; a < N; ++a)
#pragma unroll
      for (int b = 0; b < N; ++b) {
        const int o = sidx<D, N>(sR, a * SP + b * SQ);
        double dun = acc[a][b];
        if constexpr (MODE == kModeRK) dun = fma(p.rk_a, A[o], dun);
        if (!(p.dbg & 2)) {  // bit 1: timing experiment without the result stores
          __stcs(p.du + g0 + a * SP + b * SQ, dun);
          __stcs(p.out + g0 + a * SP + b * SQ, fma(p.rk_b, dun, U[o]));
        }
      }
  }
}

template <int D, int N>
__host__ __device__ constexpr int cell_smem_bytes(int CT) {
  using G = CGeo<D, N>;
  return (3 * CT * G::NDP + CT * G::FN + G::NPH * 1024 + 16) * 8 + 2 * CT * (int)sizeof(CellInfo) + 2 * (int)sizeof(UnitInfo) +
         CT * D * 16 + 16;
}

// Persistent kernel: CTA b processes units b, b + grid, ... in increasing order; each unit is GPU groups.
// Per group g: the cells of g+1 stream in (cp.async, double buffer) from g's start; g+1 is decoded at the
// start of g's last phase, its producers' flags are fetched with 16-byte cp.async (completing with g's
// epilogue) and checked after it -- so a group starts right after one barrier. The progress flag of a
// group is released by the CTA's last thread at the next group's start.
template <int D, int N, int MODE>
__global__ void __launch_bounds__(256, HD_MINB) cell_kernel(const __grid_constant__ CellParams p) {
  using G = CGeo<D, N>;
  constexpr int NPH = G::NPH;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const int CT = p.CT;
  const int CND = CT * G::NDP;
  double *smem = reinterpret_cast<double *>(smem_raw);
  // U[2] | ACC | carry[CT][FN] | ptab[NPH][4][256] | stab | info[2][CT] | uinfo[2] | fbuf[2][CT*D] (int4)
  double *ACC = smem + 2 * CND;
  double *carry0 = ACC + CND;                                  // per pencil, read before written
  double *ptab = carry0 + CT * G::FN;                          // [NPH][4][256] per-thread phase constants
  double *stab = ptab + NPH * 1024;                            // xi[8], w[8]
  CellInfo *info0 = reinterpret_cast<CellInfo *>(stab + 16);   // [2][CT]
  UnitInfo *uinfo = reinterpret_cast<UnitInfo *>(info0 + 2 * CT);  // [2]
  int4 *fbuf = reinterpret_cast<int4 *>((reinterpret_cast<uintptr_t>(uinfo + 2) + 15) & ~uintptr_t(15));
  // fbuf: [CT * D] fetched flag words (16-byte cp.async destinations)
  const int tid = threadIdx.x;
  const int k = tid / G::NT;
  const int r = tid - k * G::NT;
  const bool active = k < CT;
  if (tid < 8) {
    stab[tid] = tid < N ? c_tab[N].xi[tid] : 0.0;
    stab[8 + tid] = tid < N ? c_tab[N].w[tid] : 0.0;
  }
  if ((int)blockIdx.x >= p.nunits) return;
  phase_table<D, N, MODE>(p, r, ptab);  // read only by this thread

  // the group's cells: CT cells at cell stride cs (adjacent pencils in pencil mode, consecutive else)
  const size_t cs = p.pencil ? (size_t)p.lstride[1] : 1;
  auto copy_cells = [&](int first_cell, double *dst) {
    if constexpr (G::ND % 2 == 0) {
      for (int i = tid; i < ((CT * G::ND) >> 1); i += blockDim.x) {
        const int e = 2 * i, kc = e / G::ND, x = e - kc * G::ND;
        cp_async16(dst + kc * G::NDP + swz<D, N>(x), p.u + ((size_t)first_cell + kc * cs) * G::ND + x);
      }
    } else {
      for (int i = tid; i < CT * G::ND; i += blockDim.x) {
        const int kc = i / G::ND, x = i - kc * G::ND;
        cp_async8(dst + kc * G::NDP + swz<D, N>(x), p.u + ((size_t)first_cell + kc * cs) * G::ND + x);
      }
    }
  };
  auto first_cell = [&](int uu, int g, const UnitInfo &ui) {
    return p.pencil ? ui.base + step_group(p, g, ui.dir0, ui.skew) : uu * CT;
  };
  // decode a group into inf and fetch the flag words its publication checks need (item = (cell, dim))
  // when a group has at most one item (cell, dim) per warp (6D: one cell, 6 dims, 8 warps) the items go
  // to lane 0 of different warps, so their divergent decodes run in parallel warps instead of
  // serialising inside warp 0 (measured: 6D +1%/A +4%; with more items per warp it costs -- 5D/4D/3D)
  const int nwarps = (int)(blockDim.x >> 5);
  const int item0 = CT * D <= nwarps ? (tid >> 5) + nwarps * (tid & 31) : tid;
  auto decode_group = [&](int uu, int g, const UnitInfo &ui, CellInfo *inf) {
    for (int idx = item0; idx < CT * D; idx += (int)blockDim.x) {
      const int kk = idx / D, i = idx - kk * D;
      decode_cell<D>(p, ui, uu, g, kk, inf[kk], i);
      const int pf = inf[kk].pflag[i];
      if (pf >= 0) cp_async16(fbuf + idx, p.flags + (pf & ~3));
    }
    cp_async_commit();
  };
  auto resolve_group = [&](CellInfo *inf) {
    for (int idx = item0; idx < CT * D; idx += (int)blockDim.x) {  // same items as decode_group (own cp.async)
      const int kk = idx / D, i = idx - kk * D;
      const int pf = inf[kk].pflag[i];
      if (pf < 0) continue;
      const int4 w = fbuf[idx];
      const int q = pf & 3;
      resolve_cell(p, inf[kk], i, q == 0 ? w.x : q == 1 ? w.y : q == 2 ? w.z : w.w);
    }
  };

  int u = blockIdx.x, gi = 0, it = 0, ju = 0;
  if (p.pencil) {
    if (tid < D) decode_unit<D>(p, u, tid, uinfo[0]);
    if (tid >= 32 && tid < 32 + D && u + (int)gridDim.x < p.nunits) decode_unit<D>(p, u + gridDim.x, tid - 32, uinfo[1]);
    __syncthreads();
  }
  decode_group(u, 0, uinfo[0], info0);
  copy_cells(first_cell(u, 0, uinfo[0]), smem);
  cp_async_commit();
  cp_async_wait<0>();
  resolve_group(info0);
  int prev_unit = -1, prev_step = 0;
  while (u < p.nunits) {
    const int s = it & 1;
    CellInfo *info = info0 + s * CT;
    int un = u, gn = gi + 1;
    if (gn >= p.GPU) {
      un = u + gridDim.x;
      gn = 0;
    }
    const bool has_next = un < p.nunits;
    // group g-1 done; this group's cells, decode and flag checks are complete (waited by every thread
    // before this barrier)
    __syncthreads();
    if (prev_unit >= 0 && tid == (int)blockDim.x - 1) {
      // the previous group's traces are all written (barrier above): publish its progress
      __threadfence();
      *(volatile int *)(p.flags + prev_unit) = p.epoch | (prev_step + 1);
    }
    if (p.pencil && gi == 0 && ju > 0) {
      // decode the next unit into the slot the previous unit used
      const int u2 = u + gridDim.x;
      if (tid < D && u2 < p.nunits) decode_unit<D>(p, u2, tid, uinfo[(ju + 1) & 1]);
      if (p.GPU == 1) __syncthreads();  // needed right below by the prefetch
    }
    const UnitInfo &ui_next = uinfo[(ju + (gn == 0 ? 1 : 0)) & 1];
    if (has_next) copy_cells(first_cell(un, gn, ui_next), smem + (s ^ 1) * CND);
    cp_async_commit();
    GroupBufs gb;
    gb.U = smem + s * CND;
    gb.ACC = ACC;
    gb.carry_in = carry0 + (size_t)(active ? k : 0) * G::FN;
    gb.carry_out = carry0 + (size_t)(active ? k : 0) * G::FN;
    const CellInfo &ci = info[active ? k : 0];
    auto next_decode = [&]() {
      if (has_next) decode_group(un, gn, ui_next, info0 + (s ^ 1) * CT);
    };
    if constexpr (NPH == 1) {
      next_decode();
      run_phase<D, N, MODE, 0>(p, ci, ptab, k, r, gb, active);
    } else {
      run_phase<D, N, MODE, 0>(p, ci, ptab, k, r, gb, active);
      if constexpr (NPH == 2) {
        __syncthreads();
        next_decode();
        run_phase<D, N, MODE, (NPH > 1 ? 1 : 0)>(p, ci, ptab, k, r, gb, active);
      } else {
        __syncthreads();
        run_phase<D, N, MODE, (NPH > 1 ? 1 : 0)>(p, ci, ptab, k, r, gb, active);
        __syncthreads();
        next_decode();
        run_phase<D, N, MODE, (NPH > 2 ? 2 : 0)>(p, ci, ptab, k, r, gb, active);
      }
    }
    cp_async_wait<0>();  // next cells, next flags (and this group's dU)
    if (has_next) resolve_group(info0 + (s ^ 1) * CT);
    prev_unit = p.pubany ? u : -1;
    prev_step = gi;
    if (gn == 0) ++ju;
    u = un;
    gi = gn;
    ++it;
  }
  if (prev_unit >= 0) {
    __syncthreads();
    if (tid == (int)blockDim.x - 1) {
      __threadfence();
      *(volatile int *)(p.flags + prev_unit) = p.epoch | (prev_step + 1);
    }
  }
}

}  // namespace hd
