// hd_kernels.cu -- sm_100a FP64 kernels of the DG advection hot path.
//
// cell_kernel<D,N,MODE>: the element-centric loop of Alg. 1/Alg. 2 for one batch of
// cells per CTA iteration, persistent over batches:
//   step 1 gather      cp.async of the batch's contiguous n^d-blocks into a 128B-swizzled smem tile
//                      (double-buffered: the next batch is in flight while this one is computed)
//   step 2 cell terms  interpolation is the identity (Gauss collocation, C1); the quadrature-point
//                      operation J^-1 a |J| w_q and the gradient test are folded into
//                      1D matrices applied line by line (sum factorisation)
//   step 3 faces       upwind only needs the d upwind neighbours; the own-face
//                      term is folded into the 1D matrix; the neighbour trace (n-point dot along the
//                      normal) is read through L1/L2 and lifted with a rank-1 update
//   step 4 M^-1        exact diagonal under collocation, folded into the 1D matrices
//   step 5 scatter     coalesced stores of the cell result (+ fused LSRK update in RK mode)
// Work decomposition: dims are processed in pairs (0,1), (2,3), (4,5) (odd d: last phase has one
// active dim). In a phase a thread owns an n x n tile of the cell over the pair's two dims at fixed
// other coordinates and keeps it in registers, so both dims are contracted without smem traffic;
// the running accumulator moves between phases through a swizzled smem buffer.
#include <cuda_runtime.h>

#include <cstdio>

#include "hd_internal.h"

namespace hd {

__constant__ Tables1D c_tab[kMaxN + 1];

// ---------------------------------------------------------------------------------------------
constexpr __host__ __device__ int ipow(int b, int e) { return e == 0 ? 1 : b * ipow(b, e - 1); }
constexpr __host__ __device__ int cmin(int a, int b) { return a < b ? a : b; }
constexpr __host__ __device__ int cmax(int a, int b) { return a > b ? a : b; }

template <int D, int N>
struct Geo {
  static constexpr int ND = ipow(N, D);
  static constexpr int NT = ipow(N, D - 2);          // threads per cell
  static constexpr int NPH = (D + 1) / 2;            // phases
  static constexpr int SMEM_BUDGET = 96 * 1024;      // per CTA -> 2 CTAs per SM
  static constexpr int C = cmax(1, cmin(256 / NT, SMEM_BUDGET / (3 * ND * 8)));  // cells per batch
  static constexpr int THREADS = ((C * NT + 31) / 32) * 32;
  static constexpr int BUF = ((C * ND + 127) / 128) * 128;  // doubles, 1024-byte multiple
  static constexpr int SMEM = 3 * BUF * 8;
  static constexpr bool OK = (NT <= 1024) && (3 * ND * 8 <= 200 * 1024);
  static constexpr int MINB = SMEM <= 110 * 1024 ? 2 : 1;
  // tile dims of phase ph
  static constexpr __host__ __device__ int P(int ph) { return (D % 2 == 1 && ph == NPH - 1) ? D - 1 : 2 * ph; }
  static constexpr __host__ __device__ int Q(int ph) { return (D % 2 == 1 && ph == NPH - 1) ? D - 2 : 2 * ph + 1; }
  static constexpr __host__ __device__ bool QA(int ph) { return !(D % 2 == 1 && ph == NPH - 1); }
};

// 128B swizzle (the TMA SWIZZLE_128B pattern) on a double index within a 1024B-aligned buffer:
// the 16-byte chunk index inside each 128-byte row is XORed with (row & 7).
__device__ __forceinline__ int swz(int e) {
  const int row = e >> 4;
  return (e & ~15) | ((((e >> 1) & 7) ^ (row & 7)) << 1) | (e & 1);
}

__device__ __forceinline__ void cp_async16(void *smem_dst, const void *gsrc) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async8(void *smem_dst, const void *gsrc) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int K>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(K) : "memory"); }

__device__ __forceinline__ double ldg(const double *p) { return __ldg(p); }
__device__ __forceinline__ double2 ldg2(const double *p) { return __ldg(reinterpret_cast<const double2 *>(p)); }

// ---------------------------------------------------------------------------------------------
// Copy one batch of cells (contiguous in the vector) into a swizzled smem buffer.
template <int D, int N>
__device__ __forceinline__ void issue_batch_copy(const CellParams &p, long long batch, double *dst) {
  using G = Geo<D, N>;
  const long long first = batch * G::C;
  const long long nvalid = (p.ncells - first) < G::C ? (p.ncells - first) : G::C;
  const double *src = p.u + first * G::ND;
  const int total = (int)(nvalid * G::ND);
  if constexpr (G::ND % 2 == 0) {
    const int nch = total >> 1;
    for (int i = threadIdx.x; i < nch; i += blockDim.x) cp_async16(dst + swz(2 * i), src + 2 * i);
  } else {
    for (int i = threadIdx.x; i < total; i += blockDim.x) cp_async8(dst + swz(i), src + i);
  }
}

// Per-cell context: coordinates, upwind signs and neighbour cell indices.
template <int D>
struct CellCtx {
  long long cell;
  long long c[D];
  int sgn[D];          // 0: a_i >= 0 (left neighbour is upwind), 1: a_i < 0 (right neighbour)
  long long nb[D];     // local index of the upwind neighbour cell in dim i
};

template <int D>
__device__ __forceinline__ void cell_ctx(const CellParams &p, long long cell, CellCtx<D> &x) {
  x.cell = cell;
  long long lcx = cell % p.nx_local;
  long long cv = cell / p.nx_local;
  long long cx = p.cx_begin + lcx;
#pragma unroll
  for (int i = 0; i < D; ++i) {
    if (i < p.d_x) {
      x.c[i] = cx % p.L[i];
      cx /= p.L[i];
    } else {
      x.c[i] = cv % p.L[i];
      cv /= p.L[i];
    }
  }
#pragma unroll
  for (int i = 0; i < D; ++i) {
    double a = p.a_const[i];
#pragma unroll
    for (int j = 0; j < D; ++j) a += p.a_lin[i][j] * (p.lo[j] + ((double)x.c[j] + 0.5) * p.h[j]);
    x.sgn[i] = a < 0.0 ? 1 : 0;
    long long cn;
    if (x.sgn[i] == 0) cn = x.c[i] == 0 ? p.L[i] - 1 : x.c[i] - 1;
    else cn = x.c[i] == p.L[i] - 1 ? 0 : x.c[i] + 1;
    x.nb[i] = cell + (cn - x.c[i]) * p.lstride[i];
  }
}

// Contribution of dim P (lines along the first tile index a, indexed by b) with sign S.
//   acc[a][b] (+)= sP[b] * ( sum_j K[S][a][j] uv[j][b] + lam[S][a] * tP[b] )
template <int N, int S, bool INIT>
__device__ __forceinline__ void contrib_first(double (&acc)[N][N], const double (&uv)[N][N], const double (&tP)[N],
                                              const double (&sP)[N]) {
  const Tables1D &T = c_tab[N];
#pragma unroll
  for (int b = 0; b < N; ++b) {
#pragma unroll
    for (int a = 0; a < N; ++a) {
      double y = T.lam[S][a] * tP[b];
#pragma unroll
      for (int j = 0; j < N; ++j) y = fma(T.K[S][a][j], uv[j][b], y);
      if constexpr (INIT) acc[a][b] = sP[b] * y;
      else acc[a][b] = fma(sP[b], y, acc[a][b]);
    }
  }
}
// Contribution of dim Q (lines along the second tile index b, indexed by a).
template <int N, int S>
__device__ __forceinline__ void contrib_second(double (&acc)[N][N], const double (&uv)[N][N], const double (&tQ)[N],
                                               const double (&sQ)[N]) {
  const Tables1D &T = c_tab[N];
#pragma unroll
  for (int a = 0; a < N; ++a) {
#pragma unroll
    for (int b = 0; b < N; ++b) {
      double y = T.lam[S][b] * tQ[a];
#pragma unroll
      for (int j = 0; j < N; ++j) y = fma(T.K[S][b][j], uv[a][j], y);
      acc[a][b] = fma(sQ[a], y, acc[a][b]);
    }
  }
}

// One phase: tile dims (P, Q) at rest index r of cell slot cs.
template <int D, int N, int MODE, int PH>
__device__ __forceinline__ void run_phase(const CellParams &p, const CellCtx<D> &x, const double *U, double *ACC,
                                          int cs, int r, double (&acc)[N][N]) {
  using G = Geo<D, N>;
  constexpr int P = G::P(PH), Q = G::Q(PH);
  constexpr bool QA = G::QA(PH);
  constexpr int SP = ipow(N, P), SQ = ipow(N, Q);
  constexpr bool FIRST = PH == 0, LAST = PH == G::NPH - 1;
  const Tables1D &T = c_tab[N];

  // rest coordinates: digits of r over the dims other than P, Q (ascending)
  int mrest[D];
  int R = 0;
  {
    int rr = r;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      if (j == P || j == Q) { mrest[j] = 0; continue; }
      mrest[j] = rr % N;
      rr /= N;
      R += mrest[j] * ipow(N, j);
    }
  }
  const int ebase = cs * G::ND + R;

  // own values of the tile (registers)
  double uv[N][N];
  if constexpr (P == 0 && Q == 1 && (N % 2 == 0)) {
    // contiguous n^2 doubles: 16-byte smem loads, conflict-free under the swizzle
#pragma unroll
    for (int k = 0; k < N * N; k += 2) {
      double2 v = *reinterpret_cast<const double2 *>(U + swz(ebase + k));
      uv[k % N][k / N] = v.x;
      uv[(k + 1) % N][(k + 1) / N] = v.y;
    }
  } else {
#pragma unroll
    for (int a = 0; a < N; ++a)
#pragma unroll
      for (int b = 0; b < N; ++b) uv[a][b] = U[swz(ebase + a * SP + b * SQ)];
  }
  if constexpr (!FIRST) {
#pragma unroll
    for (int a = 0; a < N; ++a)
#pragma unroll
      for (int b = 0; b < N; ++b) acc[a][b] = ACC[swz(ebase + a * SP + b * SQ)];
  }

  // line speeds (a_i(z) / h_i) * dtfac; a_i does not depend on z_i
  double zr[D];
#pragma unroll
  for (int j = 0; j < D; ++j)
    zr[j] = (j == P || j == Q) ? 0.0 : p.lo[j] + ((double)x.c[j] + T.xi[mrest[j]]) * p.h[j];
  double sP[N], sQ[N];
  {
    double base = p.a_const[P];
#pragma unroll
    for (int j = 0; j < D; ++j)
      if (j != P && j != Q) base = fma(p.a_lin[P][j], zr[j], base);
    const double fac = p.dtfac * p.inv_h[P];
#pragma unroll
    for (int b = 0; b < N; ++b) {
      const double zq = p.lo[Q] + ((double)x.c[Q] + T.xi[b]) * p.h[Q];
      sP[b] = fma(p.a_lin[P][Q], zq, base) * fac;
    }
  }
  if constexpr (QA) {
    double base = p.a_const[Q];
#pragma unroll
    for (int j = 0; j < D; ++j)
      if (j != P && j != Q) base = fma(p.a_lin[Q][j], zr[j], base);
    const double fac = p.dtfac * p.inv_h[Q];
#pragma unroll
    for (int a = 0; a < N; ++a) {
      const double zp = p.lo[P] + ((double)x.c[P] + T.xi[a]) * p.h[P];
      sQ[a] = fma(p.a_lin[Q][P], zp, base) * fac;
    }
  }

  // upwind neighbour traces: tP[b] = sum_j tau_j u_nbP(j, b), tQ[a] = sum_j tau_j u_nbQ(a, j)
  double tP[N], tQ[N];
  {
    const double *nbP = p.u + x.nb[P] * G::ND + R;
    const int sP_ = x.sgn[P];
    double nv[N][N];
    if constexpr (P == 0 && Q == 1 && (N % 2 == 0)) {
#pragma unroll
      for (int k = 0; k < N * N; k += 2) {
        double2 v = ldg2(nbP + k);
        nv[k % N][k / N] = v.x;
        nv[(k + 1) % N][(k + 1) / N] = v.y;
      }
    } else {
#pragma unroll
      for (int j = 0; j < N; ++j)
#pragma unroll
        for (int b = 0; b < N; ++b) nv[j][b] = ldg(nbP + j * SP + b * SQ);
    }
#pragma unroll
    for (int b = 0; b < N; ++b) {
      double t = 0.0;
#pragma unroll
      for (int j = 0; j < N; ++j) t = fma(T.tau[sP_][j], nv[j][b], t);
      tP[b] = t;
    }
  }
  if constexpr (QA) {
    const double *nbQ = p.u + x.nb[Q] * G::ND + R;
    const int sQ_ = x.sgn[Q];
    double nv[N][N];
    if constexpr (P == 0 && Q == 1 && (N % 2 == 0)) {
#pragma unroll
      for (int k = 0; k < N * N; k += 2) {
        double2 v = ldg2(nbQ + k);
        nv[k % N][k / N] = v.x;
        nv[(k + 1) % N][(k + 1) / N] = v.y;
      }
    } else {
#pragma unroll
      for (int a = 0; a < N; ++a)
#pragma unroll
        for (int j = 0; j < N; ++j) nv[a][j] = ldg(nbQ + a * SP + j * SQ);
    }
#pragma unroll
    for (int a = 0; a < N; ++a) {
      double t = 0.0;
#pragma unroll
      for (int j = 0; j < N; ++j) t = fma(T.tau[sQ_][j], nv[a][j], t);
      tQ[a] = t;
    }
  }

  // contributions (sign-specialised so the 1D tables are constant-bank operands)
  if (x.sgn[P] == 0) contrib_first<N, 0, FIRST>(acc, uv, tP, sP);
  else contrib_first<N, 1, FIRST>(acc, uv, tP, sP);
  if constexpr (QA) {
    if (x.sgn[Q] == 0) contrib_second<N, 0>(acc, uv, tQ, sQ);
    else contrib_second<N, 1>(acc, uv, tQ, sQ);
  }

  if constexpr (!LAST) {
#pragma unroll
    for (int a = 0; a < N; ++a)
#pragma unroll
      for (int b = 0; b < N; ++b) ACC[swz(ebase + a * SP + b * SQ)] = acc[a][b];
  } else {
    const long long g0 = x.cell * G::ND + R;
    if constexpr (MODE == kModeAdvection) {
      // weak form: v = M (M^-1 A u), M_qq = |J| prod_i w_{q_i}
      double wr = p.jdet;
#pragma unroll
      for (int j = 0; j < D; ++j)
        if (j != P && j != Q) wr *= T.w[mrest[j]];
#pragma unroll
      for (int a = 0; a < N; ++a)
#pragma unroll
        for (int b = 0; b < N; ++b) p.out[g0 + a * SP + b * SQ] = acc[a][b] * (wr * (T.w[a] * T.w[b]));
    } else {
      // LSRK 2N stage: dU <- A_s dU + dt M^-1 A(U); U_new <- U + B_s dU
#pragma unroll
      for (int a = 0; a < N; ++a)
#pragma unroll
        for (int b = 0; b < N; ++b) {
          const long long g = g0 + a * SP + b * SQ;
          double dun = acc[a][b];
          if constexpr (MODE == kModeRK) dun = fma(p.rk_a, p.du[g], dun);
          p.du[g] = dun;
          p.out[g] = fma(p.rk_b, dun, uv[a][b]);
        }
    }
  }
}

template <int D, int N, int MODE>
__global__ void __launch_bounds__(Geo<D, N>::THREADS, Geo<D, N>::MINB) cell_kernel(const __grid_constant__ CellParams p) {
  using G = Geo<D, N>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  double *smem = reinterpret_cast<double *>(smem_raw);
  double *ACC = smem + 2 * G::BUF;
  const int tid = threadIdx.x;
  const int cs = tid / G::NT;
  const int r = tid % G::NT;

  long long b = blockIdx.x;
  if (b >= p.nbatches) return;
  issue_batch_copy<D, N>(p, b, smem);
  cp_async_commit();
  for (int it = 0; b < p.nbatches; b += gridDim.x, ++it) {
    const long long bn = b + gridDim.x;
    if (bn < p.nbatches) issue_batch_copy<D, N>(p, bn, smem + ((it + 1) & 1) * G::BUF);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const double *U = smem + (it & 1) * G::BUF;
    const long long cell = b * G::C + cs;
    const bool valid = (cs < G::C) && (cell < p.ncells);
    CellCtx<D> x;
    if (valid) cell_ctx<D>(p, cell, x);
    double acc[N][N];
    if (valid) run_phase<D, N, MODE, 0>(p, x, U, ACC, cs, r, acc);
    if constexpr (G::NPH > 1) {
      __syncthreads();
      if (valid) run_phase<D, N, MODE, (G::NPH > 1 ? 1 : 0)>(p, x, U, ACC, cs, r, acc);
    }
    if constexpr (G::NPH > 2) {
      __syncthreads();
      if (valid) run_phase<D, N, MODE, (G::NPH > 2 ? 2 : 0)>(p, x, U, ACC, cs, r, acc);
    }
    __syncthreads();
  }
  cp_async_wait<0>();
}

// ---------------------------------------------------------------------------------------------
// Streaming mass / inverse-mass kernel: u_q <- u_q * (|J| prod w)^{+-1}. The grid stride
// is a multiple of n^d so each thread's cell-local indices (and factors) are loop invariant.
template <int D, int N>
__global__ void __launch_bounds__(256) mass_kernel(const __grid_constant__ StreamParams p) {
  constexpr int ND = ipow(N, D);
  const Tables1D &T = c_tab[N];
  const long long stride = 2LL * gridDim.x * blockDim.x;
  const long long g0 = 2LL * (blockIdx.x * (long long)blockDim.x + threadIdx.x);
  double f[2];
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    int m = (int)((g0 + e) % ND);
    double w = p.jdet;
#pragma unroll
    for (int i = 0; i < D; ++i) {
      w *= T.w[m % N];
      m /= N;
    }
    f[e] = p.inverse ? 1.0 / w : w;
  }
  const long long npair = p.ndofs & ~1LL;
  long long g = g0;
  for (; g + 3 * stride < npair; g += 4 * stride) {
    double2 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = __ldcs(reinterpret_cast<const double2 *>(p.u + g + k * stride));
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      v[k].x *= f[0];
      v[k].y *= f[1];
      __stcs(reinterpret_cast<double2 *>(p.u + g + k * stride), v[k]);
    }
  }
  for (; g < npair; g += stride) {
    double2 v = __ldcs(reinterpret_cast<const double2 *>(p.u + g));
    v.x *= f[0];
    v.y *= f[1];
    __stcs(reinterpret_cast<double2 *>(p.u + g), v);
  }
  if ((p.ndofs & 1) && g0 == 0) {
    long long last = p.ndofs - 1;
    int m = (int)(last % ND);
    double w = p.jdet;
    for (int i = 0; i < D; ++i) {
      w *= T.w[m % N];
      m /= N;
    }
    p.u[last] = p.inverse ? p.u[last] / w : p.u[last] * w;
  }
}

// ---------------------------------------------------------------------------------------------
// Synthetic initial data (same recipe as paper_2002_08110_b200/inputs.py).
__device__ __forceinline__ unsigned long long splitmix64(unsigned long long z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

template <int D, int N>
__global__ void __launch_bounds__(256) fill_kernel(const __grid_constant__ FillParams p) {
  constexpr int ND = ipow(N, D);
  const Tables1D &T = c_tab[N];
  const long long total = p.ncells * ND;
  for (long long gl = blockIdx.x * (long long)blockDim.x + threadIdx.x; gl < total;
       gl += (long long)gridDim.x * blockDim.x) {
    const long long cell = gl / ND;
    int m = (int)(gl % ND);
    long long lcx = cell % p.nx_local, cv = cell / p.nx_local;
    long long cx = p.cx_begin + lcx;
    double z[D];
#pragma unroll
    for (int i = 0; i < D; ++i) {
      long long c;
      if (i < p.d_x) { c = cx % p.L[i]; cx /= p.L[i]; }
      else { c = cv % p.L[i]; cv /= p.L[i]; }
      z[i] = p.lo[i] + ((double)c + T.xi[m % N]) * p.h[i];
      m /= N;
    }
    // global DoF index (reading C19) for the counter-based generator
    long long cxg = p.cx_begin + lcx;
    long long cxtot = 1;
    for (int i = 0; i < p.d_x; ++i) cxtot *= p.L[i];
    const long long gcell = (cell / p.nx_local) * cxtot + cxg;
    const long long gg = gcell * ND + (gl % ND);
    const unsigned long long bits = splitmix64((unsigned long long)gg + (p.seed << 40));
    const double U = (double)(bits >> 11) * (1.0 / 9007199254740992.0);
    double val;
    if (p.recipe == 0) {
      const double dx = z[0] - 0.5, dy = z[1] - 0.5;
      val = exp(-(dx * dx + dy * dy) / 0.02) + (2.0 * U - 1.0) * 1e-3;
    } else if (p.recipe == 1) {
      val = 2.0 * U - 1.0;
    } else if (p.recipe == 2) {
      double pr = 1.0;
#pragma unroll
      for (int i = 0; i < D; ++i) pr *= sin(2.0 * M_PI * z[i]);
      val = pr + (2.0 * U - 1.0) * 1e-3;
    } else {
      double v2 = 0.0;
      for (int i = p.d_x; i < D; ++i) v2 += z[i] * z[i];
      val = (1.0 + 0.01 * cos(0.5 * z[0])) * pow(2.0 * M_PI, -0.5 * (D - p.d_x)) * exp(-0.5 * v2) *
            (1.0 + (2.0 * U - 1.0) * 1e-3);
    }
    p.u[gl] = val;
  }
}

// ---------------------------------------------------------------------------------------------
// Host-side dispatch over the instantiated (d, n) set.
cudaError_t upload_tables(int n, const Tables1D &t) {
  return cudaMemcpyToSymbol(c_tab, &t, sizeof(Tables1D), sizeof(Tables1D) * n, cudaMemcpyHostToDevice);
}

namespace {

template <int D, int N, int MODE>
cudaError_t launch_cell_impl(const CellParams &p, cudaStream_t s, int sms) {
  using G = Geo<D, N>;
  static int occ = -1;
  auto kern = cell_kernel<D, N, MODE>;
  if (occ < 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, G::THREADS, G::SMEM);
    if (e != cudaSuccess) return e;
    if (occ < 1) occ = 1;
  }
  long long grid = (long long)sms * occ;
  if (grid > p.nbatches) grid = p.nbatches;
  if (grid < 1) return cudaSuccess;
  kern<<<(unsigned)grid, G::THREADS, G::SMEM, s>>>(p);
  return cudaGetLastError();
}

template <int D, int N>
cudaError_t launch_cell_dn(const CellParams &p, cudaStream_t s, int sms) {
  if constexpr (!Geo<D, N>::OK) {
    return cudaErrorNotSupported;
  } else {
    switch (p.mode) {
      case kModeAdvection: return launch_cell_impl<D, N, kModeAdvection>(p, s, sms);
      case kModeRK: return launch_cell_impl<D, N, kModeRK>(p, s, sms);
      default: return launch_cell_impl<D, N, kModeRKFirst>(p, s, sms);
    }
  }
}

template <int D, int N>
cudaError_t launch_mass_dn(const StreamParams &p, cudaStream_t s, int sms) {
  constexpr int ND = ipow(N, D);
  // grid * 512 must be a multiple of ND (loop-invariant local indices)
  long long g0 = ND;
  {
    long long a = ND, b = 512;
    while (b) { long long t = a % b; a = b; b = t; }
    g0 = ND / a;
  }
  long long want = (long long)sms * 8;
  long long grid = ((want + g0 - 1) / g0) * g0;
  long long need = (p.ndofs / 2 + 255) / 256;  // no more blocks than pairs need
  if (need < 1) need = 1;
  long long cap = ((need + g0 - 1) / g0) * g0;
  if (grid > cap) grid = cap;
  mass_kernel<D, N><<<(unsigned)grid, 256, 0, s>>>(p);
  return cudaGetLastError();
}

template <int D, int N>
cudaError_t launch_fill_dn(const FillParams &p, cudaStream_t s) {
  long long total = p.ncells * (long long)ipow(N, D);
  long long grid = (total + 255) / 256;
  if (grid > 148LL * 64) grid = 148LL * 64;
  if (grid < 1) grid = 1;
  fill_kernel<D, N><<<(unsigned)grid, 256, 0, s>>>(p);
  return cudaGetLastError();
}

#define HD_DISPATCH_N(D, FN, ...)                  \
  switch (n) {                                     \
    case 2: return FN<D, 2>(__VA_ARGS__);          \
    case 3: return FN<D, 3>(__VA_ARGS__);          \
    case 4: return FN<D, 4>(__VA_ARGS__);          \
    case 5: return FN<D, 5>(__VA_ARGS__);          \
    case 6: return FN<D, 6>(__VA_ARGS__);          \
    default: return cudaErrorNotSupported;         \
  }
#define HD_DISPATCH(FN, ...)                       \
  switch (d) {                                     \
    case 2: HD_DISPATCH_N(2, FN, __VA_ARGS__)      \
    case 3: HD_DISPATCH_N(3, FN, __VA_ARGS__)      \
    case 4: HD_DISPATCH_N(4, FN, __VA_ARGS__)      \
    case 5: HD_DISPATCH_N(5, FN, __VA_ARGS__)      \
    case 6: HD_DISPATCH_N(6, FN, __VA_ARGS__)      \
    default: return cudaErrorNotSupported;         \
  }

template <int D, int N>
bool supported_dn() { return Geo<D, N>::OK; }
template <int D, int N>
int cpb_dn() { return Geo<D, N>::C; }

}  // namespace

cudaError_t launch_cell_kernel(int d, int n, const CellParams &p, cudaStream_t s, long long *launches, int sms) {
  if (launches) ++*launches;
  HD_DISPATCH(launch_cell_dn, p, s, sms)
}
cudaError_t launch_mass_kernel(int d, int n, const StreamParams &p, cudaStream_t s, long long *launches, int sms) {
  if (launches) ++*launches;
  HD_DISPATCH(launch_mass_dn, p, s, sms)
}
cudaError_t launch_fill_kernel(int d, int n, const FillParams &p, cudaStream_t s, long long *launches) {
  if (launches) ++*launches;
  HD_DISPATCH(launch_fill_dn, p, s)
}

bool cell_kernel_supported(int d, int n) {
  if (d < 2 || d > 6 || n < 2 || n > 6) return false;
  switch (d) {
    case 2: switch (n) { case 2: return supported_dn<2, 2>(); case 3: return supported_dn<2, 3>(); case 4: return supported_dn<2, 4>(); case 5: return supported_dn<2, 5>(); default: return supported_dn<2, 6>(); }
    case 3: switch (n) { case 2: return supported_dn<3, 2>(); case 3: return supported_dn<3, 3>(); case 4: return supported_dn<3, 4>(); case 5: return supported_dn<3, 5>(); default: return supported_dn<3, 6>(); }
    case 4: switch (n) { case 2: return supported_dn<4, 2>(); case 3: return supported_dn<4, 3>(); case 4: return supported_dn<4, 4>(); case 5: return supported_dn<4, 5>(); default: return supported_dn<4, 6>(); }
    case 5: switch (n) { case 2: return supported_dn<5, 2>(); case 3: return supported_dn<5, 3>(); case 4: return supported_dn<5, 4>(); case 5: return supported_dn<5, 5>(); default: return supported_dn<5, 6>(); }
    default: switch (n) { case 2: return supported_dn<6, 2>(); case 3: return supported_dn<6, 3>(); case 4: return supported_dn<6, 4>(); case 5: return supported_dn<6, 5>(); default: return supported_dn<6, 6>(); }
  }
}

int cells_per_batch(int d, int n) {
  switch (d) {
    case 2: switch (n) { case 2: return cpb_dn<2, 2>(); case 3: return cpb_dn<2, 3>(); case 4: return cpb_dn<2, 4>(); case 5: return cpb_dn<2, 5>(); default: return cpb_dn<2, 6>(); }
    case 3: switch (n) { case 2: return cpb_dn<3, 2>(); case 3: return cpb_dn<3, 3>(); case 4: return cpb_dn<3, 4>(); case 5: return cpb_dn<3, 5>(); default: return cpb_dn<3, 6>(); }
    case 4: switch (n) { case 2: return cpb_dn<4, 2>(); case 3: return cpb_dn<4, 3>(); case 4: return cpb_dn<4, 4>(); case 5: return cpb_dn<4, 5>(); default: return cpb_dn<4, 6>(); }
    case 5: switch (n) { case 2: return cpb_dn<5, 2>(); case 3: return cpb_dn<5, 3>(); case 4: return cpb_dn<5, 4>(); case 5: return cpb_dn<5, 5>(); default: return cpb_dn<5, 6>(); }
    default: switch (n) { case 2: return cpb_dn<6, 2>(); case 3: return cpb_dn<6, 3>(); case 4: return cpb_dn<6, 4>(); case 5: return cpb_dn<6, 5>(); default: return cpb_dn<6, 6>(); }
  }
}

}  // namespace hd
