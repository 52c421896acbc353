// hd_basis.cu -- basis change between the GLL nodal basis and the Gauss-point values (SURVEY §8(f) NEXT-2,
// Cartesian part; "a sequence of d 1D interpolation sweeps"; DESIGN.md §6
// "Basis change").
//
//   basis_kernel<N>: v_cell <- (S x ... x S) u_cell for every cell, S the n x n matrix of one hd_basis_kind.
//
// HBM-bound by design (16 B/DoF: every value read once, written once). A CTA stages a batch of whole cells
// (>= 4096 doubles where the mesh has them) in shared memory, then applies the d sweeps two dims at a time:
// a thread owns an N x N tile over dims (i, i+1), contracts both in registers and writes it back in place, so
// a value crosses shared memory ceil(d/2) times instead of d. Cells are contiguous blocks of N^d values, so
// the tile index runs over the whole batch (the cell index is part of its high digits). The staging buffer
// carries one pad double per 32 (tiles of the first pass are 16 contiguous doubles per thread).
#include <cuda_runtime.h>

#include "hd_internal.h"

namespace hd {

namespace {

__device__ __forceinline__ int padded(int x) { return x + (x >> 5); }

template <int N>
__global__ void __launch_bounds__(256) basis_kernel(const __grid_constant__ BasisParams p) {
  extern __shared__ double sm[];
  int ND = 1;
  for (int i = 0; i < p.d; ++i) ND *= N;
  const long long nb = (p.ncells + p.cb - 1) / p.cb;
  for (long long b = blockIdx.x; b < nb; b += gridDim.x) {
    const long long c0 = b * p.cb;
    const long long left = p.ncells - c0;
    const int cnt = (int)(left < p.cb ? left : p.cb) * ND;
    const double *src = p.u + c0 * ND;
    double *dst = p.v + c0 * ND;
    __syncthreads();  // the previous batch's copy-out has read the buffer
    if constexpr (N % 2 == 0) {  // ND even: 16-B aligned batches
      for (int e = 2 * threadIdx.x; e < cnt; e += 2 * blockDim.x) {
        const double2 x = __ldcs(reinterpret_cast<const double2 *>(src + e));
        sm[padded(e)] = x.x;
        sm[padded(e + 1)] = x.y;
      }
    } else {
      for (int e = threadIdx.x; e < cnt; e += blockDim.x) sm[padded(e)] = __ldcs(src + e);
    }
    __syncthreads();
    int st = 1;  // N^i
    int i = 0;
    for (; i + 1 < p.d; i += 2) {  // dims (i, i+1) together
      const int nt = cnt / (N * N);
      for (int l = threadIdx.x; l < nt; l += blockDim.x) {
        const int lo = l % st, hi = l / st;
        const int base = hi * st * N * N + lo;
        double x[N][N], y[N][N];
#pragma unroll
        for (int q1 = 0; q1 < N; ++q1)
#pragma unroll
          for (int q0 = 0; q0 < N; ++q0) x[q1][q0] = sm[padded(base + (q0 + N * q1) * st)];
#pragma unroll
        for (int q1 = 0; q1 < N; ++q1)
#pragma unroll
          for (int m0 = 0; m0 < N; ++m0) {
            double s = 0.0;
#pragma unroll
            for (int q0 = 0; q0 < N; ++q0) s = fma(p.S[m0 * N + q0], x[q1][q0], s);
            y[q1][m0] = s;
          }
#pragma unroll
        for (int m1 = 0; m1 < N; ++m1)
#pragma unroll
          for (int m0 = 0; m0 < N; ++m0) {
            double s = 0.0;
#pragma unroll
            for (int q1 = 0; q1 < N; ++q1) s = fma(p.S[m1 * N + q1], y[q1][m0], s);
            sm[padded(base + (m0 + N * m1) * st)] = s;
          }
      }
      st *= N * N;
      __syncthreads();
    }
    if (i < p.d) {  // odd d: the last dim alone
      const int nl = cnt / N;
      for (int l = threadIdx.x; l < nl; l += blockDim.x) {
        const int lo = l % st, hi = l / st;
        const int base = hi * st * N + lo;
        double x[N];
#pragma unroll
        for (int q = 0; q < N; ++q) x[q] = sm[padded(base + q * st)];
#pragma unroll
        for (int m = 0; m < N; ++m) {
          double s = 0.0;
#pragma unroll
          for (int q = 0; q < N; ++q) s = fma(p.S[m * N + q], x[q], s);
          sm[padded(base + m * st)] = s;
        }
      }
      __syncthreads();
    }
    if constexpr (N % 2 == 0) {
      for (int e = 2 * threadIdx.x; e < cnt; e += 2 * blockDim.x)
        __stcs(reinterpret_cast<double2 *>(dst + e), make_double2(sm[padded(e)], sm[padded(e + 1)]));
    } else {
      for (int e = threadIdx.x; e < cnt; e += blockDim.x) __stcs(dst + e, sm[padded(e)]);
    }
  }
}

constexpr int kBatchDoubles = 4096;
constexpr size_t kMaxSmem = 200 * 1024;

long long ipow_ll(int b, int e) {
  long long r = 1;
  for (int i = 0; i < e; ++i) r *= b;
  return r;
}

size_t smem_of(long long doubles) { return (size_t)(doubles + doubles / 32 + 1) * sizeof(double); }

template <int N>
cudaError_t launch_n(BasisParams &p, cudaStream_t s, int sms) {
  const long long ND = ipow_ll(N, p.d);
  long long cb = kBatchDoubles / ND;
  if (cb < 1) cb = 1;
  if (cb > p.ncells) cb = p.ncells;
  p.cb = (int)cb;
  const size_t smem = smem_of(cb * ND);
  cudaError_t e = cudaFuncSetAttribute(basis_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxSmem);
  if (e != cudaSuccess) return e;
  const long long nb = (p.ncells + cb - 1) / cb;
  int per_sm = (int)(kMaxSmem / (smem + 1024));
  if (per_sm > 8) per_sm = 8;
  if (per_sm < 1) per_sm = 1;
  const long long cap = (long long)sms * per_sm;
  basis_kernel<N><<<(unsigned)(nb < cap ? nb : cap), 256, smem, s>>>(p);
  return cudaGetLastError();
}

}  // namespace

bool basis_kernel_supported(int d, int n) {
  return d >= 1 && d <= 6 && n >= 2 && n <= kMaxN && smem_of(ipow_ll(n, d)) <= kMaxSmem;
}

cudaError_t launch_basis_kernel(int n, BasisParams &p, cudaStream_t s, long long *launches, int sms) {
  if (p.ncells <= 0) return cudaSuccess;
  if (launches) ++*launches;
  switch (n) {
    case 2: return launch_n<2>(p, s, sms);
    case 3: return launch_n<3>(p, s, sms);
    case 4: return launch_n<4>(p, s, sms);
    case 5: return launch_n<5>(p, s, sms);
    case 6: return launch_n<6>(p, s, sms);
    default: break;
  }
  return cudaErrorNotSupported;
}

}  // namespace hd
