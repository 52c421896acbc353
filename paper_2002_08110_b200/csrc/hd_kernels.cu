// hd_kernels.cu -- sm_100a FP64 kernels of the DG advection hot path and their dispatch.
//
//   cell_kernel<D,N,MODE> (hd_cell.cuh)  the fused element-centric loop of Alg. 1/Alg. 2:
//                                        A, M^-1 A and the LSRK stage in one persistent kernel
//   mass_kernel<D,N>                     stand-alone u <- M^-1 u / M u
//   fill_kernel<D,N>                     seeded synthetic initial data
//   pack_kernel<D,N>                     outgoing halo traces of a rank
// Instantiated for d = 2..6 and n = 2..6 where one cell fits the kernel (CGeo::OK); the host picks the
// group geometry (cells per group, pencil mode) per mesh.
#include <cuda_runtime.h>

#include <cstdio>
#include <type_traits>

#include "hd_internal.h"

namespace hd {

__constant__ Tables1D c_tab[kMaxN + 1];

// ---------------------------------------------------------------------------------------------
constexpr __host__ __device__ int ipow(int b, int e) { return e == 0 ? 1 : b * ipow(b, e - 1); }
constexpr __host__ __device__ int cmin(int a, int b) { return a < b ? a : b; }
constexpr __host__ __device__ int cmax(int a, int b) { return a > b ? a : b; }

__device__ __forceinline__ void cp_async16(void *smem_dst, const void *gsrc) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async8(void *smem_dst, const void *gsrc) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gsrc) : "memory");
}
// 16-byte cp.async with an L2 eviction-priority policy (createpolicy: evict_first for data read once)
__device__ __forceinline__ unsigned long long l2_policy_evict_first() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void cp_async16_hint(void *smem_dst, const void *gsrc, unsigned long long pol) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gsrc), "l"(pol) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int K>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(K) : "memory"); }

}  // namespace hd

#include "hd_cell.cuh"

namespace hd {

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
    long long cell = gl / ND;
    const int m0 = (int)(gl % ND);
    int m = m0;
    double z[D];
    long long gcell = 0, gs = 1;
#pragma unroll
    for (int i = 0; i < D; ++i) {
      const long long c = p.off[i] + cell % p.len[i];  // global cell coordinate
      cell /= p.len[i];
      z[i] = p.lo[i] + ((double)c + T.xi[m % N]) * p.h[i];
      m /= N;
      gcell += c * gs;
      gs *= p.L[i];
    }
    // global DoF index (reading C19) for the counter-based generator
    const long long gg = gcell * ND + m0;
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
// Halo pack: the (scaled) downwind trace of each listed cell along its listed dim, written in
// the consumer's phase layout (face point f = N r + l: rest digits r, partner tile digit l). The line speed
// and the trace are evaluated with the cell kernel's expressions (line_speed, line_trace), so a trace that
// crosses ranks has the bits it would have had inside one rank.
template <int D, int N>
__device__ __forceinline__ double pack_cell_base(const CellParams &p, int X, long long cell) {
  double ab = p.a_const[X];
#pragma unroll
  for (int j = 0; j < D; ++j) {
    const long long c = cell % p.L[j];
    cell /= p.L[j];
    ab = fma(p.a_lin[X][j], fma((double)((int)c + p.coff[j]), p.h[j], p.lo[j]), ab);
  }
  return ab;
}

template <int D, int N>
__global__ void __launch_bounds__(256) pack_kernel(const __grid_constant__ PackParams pp, const __grid_constant__ CellParams p) {
  using G = CGeo<D, N>;
  const long long total = pp.nent * G::FN;
  for (long long gi = blockIdx.x * (long long)blockDim.x + threadIdx.x; gi < total;
       gi += (long long)gridDim.x * blockDim.x) {
    const long long e = gi / G::FN;
    const int f = (int)(gi - e * G::FN);
    const int ds = pp.dimsg[e];
    const int X = ds & 255, S = ds >> 8;
    // the consumer's phase of dim X, partner dim Y, rest index r and partner digit l of face point f
    const int ph = (X == 0 || X == D - 1) ? 0 : (X + 1) / 2;
    const int P = G::P(ph), Q = G::Q(ph);
    const int Y = X == P ? Q : P;
    const int r = f / N, l = f - r * N;
    // rest offset of the speed (thread_phase's sum, same order)
    double w = 0.0;
    int rr = r;
    for (int j = 0; j < D; ++j) {
      if (j != P && j != Q) {
        const int m = rr % N;
        rr /= N;
        w = fma(p.a_lin[X][j] * p.h[j], c_tab[N].xi[m], w);
      }
    }
    const LineSpeed ls = line_speed(p, X, Y, pack_cell_base<D, N>(p, X, pp.cells[e]), w);
    const double s = p.var[X] ? fma(ls.sl, c_tab[N].xi[l], ls.s0) : 0.0;
    int sx = 1;
    for (int j = 0; j < X; ++j) sx *= N;
    const double *src = pp.u + (size_t)pp.cells[e] * G::ND + face_offset<D, N>(X, f);
    // line_trace with a run-time dim
    double us[N];
#pragma unroll
    for (int j = 0; j < N; ++j) {
      const double v = __ldg(src + j * sx);
      us[j] = p.var[X] ? s * v : v;
    }
    const double *tau = p.var[X] ? c_tab[N].tau[S] : p.Ts + (X * 2 + S) * N;
    double t = tau[0] * us[0];
#pragma unroll
    for (int j = 1; j < N; ++j) t = fma(tau[j], us[j], t);
    pp.out[gi] = t;
#ifdef HD_DEBUG
    if (f == 0) p.stag[X * 2 + S] = p.epoch;  // freshness tag of this stage's traces
#endif
  }
}

// HD_DEBUG: non-finite values after an RK stage
__global__ void __launch_bounds__(256) finite_kernel(const double *v, long long n, int *err) {
  int bad = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    bad |= !isfinite(v[i]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(err, 4);
}

// ---------------------------------------------------------------------------------------------
// Host-side dispatch over the instantiated (d, n) set.
cudaError_t upload_tables(int n, const Tables1D &t) {
  return cudaMemcpyToSymbol(c_tab, &t, sizeof(Tables1D), sizeof(Tables1D) * n, cudaMemcpyHostToDevice);
}

namespace {

// Kernel instances built: every (d, n) whose cell fits (CGeo::OK). HD_ONLY_BENCH (experiment builds,
// `python -m paper_2002_08110_b200.build -DHD_ONLY_BENCH --out=...`) keeps only the bench configs.
template <int D, int N>
constexpr bool built() {
#ifdef HD_ONLY_BENCH
  if (!((D == 4 && N == 4) || (D == 5 && N == 4) || (D == 6 && N == 4) || (D == 3 && N == 5))) return false;
#endif
  return CGeo<D, N>::OK;
}

template <int D, int N>
CellGeometry geometry_dn(int L0, int L1, long long ncells, int pencil_ok) {
  using G = CGeo<D, N>;
  CellGeometry g{};
  g.phases = G::NPH;
  // the kernel lays out max_ct cells (compile-time smem offsets); any group up to that size fits
  const int maxCT = max_ct<D, N>();
  const int kSmemMax = 227 * 1024;
  auto smem_of = [&](int) { return cell_smem_bytes<D, N>(); };
  if (L0 <= maxCT && smem_of(L0) <= kSmemMax) {
    // multi-pencil groups: m whole pencils per group
    const long long npen = ncells / L0;
    int m = 1;
    for (int c = 1; c * L0 <= maxCT; ++c)
      if (npen % c == 0 && smem_of(c * L0) <= kSmemMax) m = c;
    g.CT = m * L0;
    g.pencil = 0;
    g.GPU = 1;
  } else if (!pencil_ok) {
    // chunk mode (a_0 depends on z_1, so the pencils of a pencil-mode group would sweep dim 0 in
    // different directions): a group is CT consecutive cells of one pencil (CT | L0); dim-0 neighbours
    // outside the group are read directly
    int CT = 1;
    for (int c = 1; c <= maxCT; ++c)
      if (L0 % c == 0 && smem_of(c) <= kSmemMax) CT = c;
    g.CT = CT;
    g.pencil = 0;
    g.GPU = 1;
  } else {
    // pencil mode: a group is CT cells from CT adjacent pencils (CT | L1), one group per dim-0 position
    int CT = 1;
    for (int c = 1; c <= maxCT; ++c)
      if (L1 % c == 0 && smem_of(c) <= kSmemMax) CT = c;
    g.CT = CT;
    g.pencil = 1;
    g.GPU = L0;
  }
  g.threads = ((g.CT * G::NT + 31) / 32) * 32;
  g.smem = cell_smem_bytes<D, N>();
  return g;
}

template <int D, int N, int MODE>
cudaError_t grid_impl(const CellGeometry &g, int sms, int *grid) {
  auto kern = cell_kernel<D, N, MODE>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  if (e != cudaSuccess) return e;
  int occ = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, g.threads, g.smem);
  if (e != cudaSuccess) return e;
  *grid = (occ < 1 ? 1 : occ) * sms;
  return cudaSuccess;
}

template <int D, int N, int MODE>
cudaError_t launch_cell_impl(const CellParams &p, cudaStream_t s, int grid_max) {
  // the host decided the geometry (hd_create_mesh); only the block size and smem follow from it
  const int threads = ((p.CT * CGeo<D, N>::NT + 31) / 32) * 32;
  const int smem = cell_smem_bytes<D, N>();
  const int nu = p.u_end - p.u_begin;
  int grid = grid_max < nu ? grid_max : nu;
  if (grid < 1) return cudaSuccess;
  cell_kernel<D, N, MODE><<<grid, threads, smem, s>>>(p);
  return cudaGetLastError();
}

template <int D, int N>
cudaError_t launch_cell_dn(const CellParams &p, cudaStream_t s, int grid_max) {
  if constexpr (!built<D, N>()) {
    return cudaErrorNotSupported;
  } else {
    switch (p.mode) {
      case kModeAdvection: return launch_cell_impl<D, N, kModeAdvection>(p, s, grid_max);
      case kModeRK: return launch_cell_impl<D, N, kModeRK>(p, s, grid_max);
      case kModeAdvAcc: return launch_cell_impl<D, N, kModeAdvAcc>(p, s, grid_max);
      default: return launch_cell_impl<D, N, kModeRKFirst>(p, s, grid_max);
    }
  }
}

template <int D, int N>
cudaError_t grid_dn(const CellGeometry &g, int sms, int *grid) {
  if constexpr (!built<D, N>()) {
    return cudaErrorNotSupported;
  } else {
    // all modes share the geometry; take the minimum co-residency over them
    int g0 = 0, g1 = 0, g2 = 0, g3 = 0;
    cudaError_t e = grid_impl<D, N, kModeAdvection>(g, sms, &g0);
    if (e == cudaSuccess) e = grid_impl<D, N, kModeRK>(g, sms, &g1);
    if (e == cudaSuccess) e = grid_impl<D, N, kModeRKFirst>(g, sms, &g2);
    if (e == cudaSuccess) e = grid_impl<D, N, kModeAdvAcc>(g, sms, &g3);
    int m = g0 < g1 ? g0 : g1;
    m = m < g2 ? m : g2;
    *grid = m < g3 ? m : g3;
    return e;
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
  long long need = (p.ndofs / 2 + 255) / 256;
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

template <int D, int N>
cudaError_t launch_pack_dn(const PackParams &pp, const CellParams &p, cudaStream_t s) {
  long long total = pp.nent * (long long)ipow(N, D - 1);
  long long grid = (total + 255) / 256;
  if (grid > 148LL * 16) grid = 148LL * 16;
  if (grid < 1) return cudaSuccess;
  pack_kernel<D, N><<<(unsigned)grid, 256, 0, s>>>(pp, p);
  return cudaGetLastError();
}

template <int D, int N>
bool supported_dn() { return built<D, N>(); }

#define HD_DISPATCH_N(D, FN, ...)                  \
  switch (n) {                                     \
    case 2: return FN<D, 2>(__VA_ARGS__);          \
    case 3: return FN<D, 3>(__VA_ARGS__);          \
    case 4: return FN<D, 4>(__VA_ARGS__);          \
    case 5: return FN<D, 5>(__VA_ARGS__);          \
    case 6: return FN<D, 6>(__VA_ARGS__);          \
    default: break;                                \
  }                                                \
  break;
#define HD_DISPATCH(FN, FAIL, ...)                 \
  switch (d) {                                     \
    case 2: HD_DISPATCH_N(2, FN, __VA_ARGS__)      \
    case 3: HD_DISPATCH_N(3, FN, __VA_ARGS__)      \
    case 4: HD_DISPATCH_N(4, FN, __VA_ARGS__)      \
    case 5: HD_DISPATCH_N(5, FN, __VA_ARGS__)      \
    case 6: HD_DISPATCH_N(6, FN, __VA_ARGS__)      \
    default: break;                                \
  }                                                \
  return FAIL;

}  // namespace

cudaError_t launch_cell_kernel(int d, int n, const CellParams &p, cudaStream_t s, long long *launches, int grid) {
  if (launches) ++*launches;
  HD_DISPATCH(launch_cell_dn, cudaErrorNotSupported, p, s, grid)
}
cudaError_t launch_mass_kernel(int d, int n, const StreamParams &p, cudaStream_t s, long long *launches, int sms) {
  if (launches) ++*launches;
  HD_DISPATCH(launch_mass_dn, cudaErrorNotSupported, p, s, sms)
}
cudaError_t launch_fill_kernel(int d, int n, const FillParams &p, cudaStream_t s, long long *launches) {
  if (launches) ++*launches;
  HD_DISPATCH(launch_fill_dn, cudaErrorNotSupported, p, s)
}
cudaError_t launch_pack_kernel(int d, int n, const PackParams &pp, const CellParams &cp, cudaStream_t s,
                               long long *launches) {
  if (launches) ++*launches;
  HD_DISPATCH(launch_pack_dn, cudaErrorNotSupported, pp, cp, s)
}
bool cell_kernel_supported(int d, int n) { HD_DISPATCH(supported_dn, false) }
cudaError_t launch_finite_check(const double *v, long long n, int *err, cudaStream_t s) {
  finite_kernel<<<148 * 8, 256, 0, s>>>(v, n, err);
  return cudaGetLastError();
}
CellGeometry cell_geometry(int d, int n, int L0, int L1, long long ncells, int pencil_ok) {
  HD_DISPATCH(geometry_dn, CellGeometry{}, L0, L1, ncells, pencil_ok)
}
cudaError_t cell_grid_size(int d, int n, const CellGeometry &g, int sms, int *grid) {
  HD_DISPATCH(grid_dn, cudaErrorNotSupported, g, sms, grid)
}

}  // namespace hd
