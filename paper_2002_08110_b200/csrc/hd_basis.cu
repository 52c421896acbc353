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
// is padded (see padded<N>) so that the per-thread contiguous tiles of the first pass do not collide in banks. Persistent
// CTAs (as many as stay resident) with two staging buffers: the next batch arrives by cp.async while the
// current one is contracted and streamed out (one buffer where two do not fit).
#include <cuda_runtime.h>

#include "hd_internal.h"

namespace hd {

namespace {

// Staging-buffer index of value x. Even n: two pad doubles per 16 -- keeps every even index 16-byte aligned (16-byte
// cp.async, LDS.128 / STS.128 in the first pass and the read-out) and is conflict-free for the 16-double tiles of
// the first pass read as 16-byte words as well as for the strided 8-byte accesses of the later passes. Odd n: one
// pad double per 32, 8-byte accesses throughout.
template <int N>
__device__ __forceinline__ int padded(int x) {
  return (N % 2 == 0) ? x + 2 * (x >> 4) : x + (x >> 5);
}

// dims (i, i+1) of every tile of the batch, ST = N^i: x <- (S x S) x in place
template <int N, int ST>
__device__ __forceinline__ void tile_pass(double *sm, int cnt, const double *S) {
  const int nt = cnt / (N * N);
  for (int l = threadIdx.x; l < nt; l += blockDim.x) {
    const int lo = l % ST, hi = l / ST;
    const int base = hi * (ST * N * N) + lo;
    constexpr bool kVec = ST == 1 && N % 2 == 0;  // the tile is N^2 contiguous doubles starting at an even index
    // tile elements a multiple of 16 apart from a base (or, first pass, inside one aligned 16-block): the padded
    // index is padded(base) plus a compile-time offset, so the accesses use immediate offsets
    constexpr bool kConst = N % 2 == 0 && (ST % 16 == 0 || (ST == 1 && N * N == 16));
    const int pb = padded<N>(base);
    auto at = [&](int off) { return kConst ? pb + off + 2 * (off >> 4) : padded<N>(base + off); };
    double x[N][N];
    if constexpr (kVec) {
#pragma unroll
      for (int q = 0; q < N * N; q += 2) {
        const double2 v = *reinterpret_cast<const double2 *>(&sm[at(q)]);
        x[q / N][q % N] = v.x;
        x[(q + 1) / N][(q + 1) % N] = v.y;
      }
    } else {
#pragma unroll
      for (int q1 = 0; q1 < N; ++q1)
#pragma unroll
        for (int q0 = 0; q0 < N; ++q0) x[q1][q0] = sm[at((q0 + N * q1) * ST)];
    }
#pragma unroll
    for (int q1 = 0; q1 < N; ++q1) {  // dim i, row by row in place
      double t[N];
#pragma unroll
      for (int m0 = 0; m0 < N; ++m0) {
        double a = 0.0;
#pragma unroll
        for (int q0 = 0; q0 < N; ++q0) a = fma(S[m0 * N + q0], x[q1][q0], a);
        t[m0] = a;
      }
#pragma unroll
      for (int m0 = 0; m0 < N; ++m0) x[q1][m0] = t[m0];
    }
    if constexpr (kVec) {  // dim i+1, two neighbouring columns at a time, 16-byte stores
#pragma unroll
      for (int m1 = 0; m1 < N; ++m1)
#pragma unroll
        for (int m0 = 0; m0 < N; m0 += 2) {
          double a = 0.0, c = 0.0;
#pragma unroll
          for (int q1 = 0; q1 < N; ++q1) {
            a = fma(S[m1 * N + q1], x[q1][m0], a);
            c = fma(S[m1 * N + q1], x[q1][m0 + 1], c);
          }
          *reinterpret_cast<double2 *>(&sm[at(m0 + N * m1)]) = make_double2(a, c);
        }
    } else {
#pragma unroll
      for (int m0 = 0; m0 < N; ++m0)  // dim i+1, column by column straight to shared memory
#pragma unroll
        for (int m1 = 0; m1 < N; ++m1) {
          double a = 0.0;
#pragma unroll
          for (int q1 = 0; q1 < N; ++q1) a = fma(S[m1 * N + q1], x[q1][m0], a);
          sm[at((m0 + N * m1) * ST)] = a;
        }
    }
  }
}

// the last dim of an odd d alone, ST = N^(d-1)
template <int N, int ST>
__device__ __forceinline__ void line_pass(double *sm, int cnt, const double *S) {
  const int nl = cnt / N;
  for (int l = threadIdx.x; l < nl; l += blockDim.x) {
    const int lo = l % ST, hi = l / ST;
    const int base = hi * (ST * N) + lo;
    double x[N];
#pragma unroll
    for (int q = 0; q < N; ++q) x[q] = sm[padded<N>(base + q * ST)];
#pragma unroll
    for (int m = 0; m < N; ++m) {
      double a = 0.0;
#pragma unroll
      for (int q = 0; q < N; ++q) a = fma(S[m * N + q], x[q], a);
      sm[padded<N>(base + m * ST)] = a;
    }
  }
}

__device__ __forceinline__ void cp_async8(void *smem_dst, const void *gsrc) {
  unsigned a = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(a), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async16(void *smem_dst, const void *gsrc) {
  unsigned a = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(a), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int K>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(K) : "memory"); }

template <int N>
__global__ void __launch_bounds__(256, N <= 3 ? 4 : N == 4 ? 3 : N == 5 ? 2 : 1)
    basis_kernel(const __grid_constant__ BasisParams p) {
  extern __shared__ __align__(16) double smem[];
  constexpr int N2 = N * N, N4 = N2 * N2;
  int ND = 1;
  for (int i = 0; i < p.d; ++i) ND *= N;
  const long long nb = (p.ncells + p.cb - 1) / p.cb;
  const int full = p.cb * ND;
  const int bufsz = (N % 2 == 0) ? full + 2 * (full >> 4) + 2 : full + (full >> 5) + 1;  // padded doubles per buffer
  auto count_of = [&](long long b) {
    const long long left = p.ncells - b * p.cb;
    return (int)(left < p.cb ? left : p.cb) * ND;
  };
  // stage batch b by cp.async (16 bytes for even n, where batches and padded even indices are 16-byte aligned;
  // 8 bytes for odd n): all of a thread's copies in flight at once and none held in registers
  auto issue = [&](long long b, double *buf) {
    const double *src = p.u + b * (long long)full;
    const int cnt = count_of(b);
    if constexpr (N % 2 == 0) {
      for (int e = 2 * threadIdx.x; e < cnt; e += 2 * blockDim.x) cp_async16(buf + padded<N>(e), src + e);
    } else {
      for (int e = threadIdx.x; e < cnt; e += blockDim.x) cp_async8(buf + padded<N>(e), src + e);
    }
  };
  long long b = blockIdx.x;
  int cur = 0;
  if (b < nb) issue(b, smem);
  cp_async_commit();
  for (; b < nb; b += gridDim.x) {
    const long long nxt = b + gridDim.x;
    double *sm = smem + cur * bufsz;
    if (p.nbuf == 2) {  // the next batch streams in while this one is contracted and written out
      if (nxt < nb) issue(nxt, smem + (cur ^ 1) * bufsz);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const int cnt = count_of(b);
    if (p.d >= 2) { tile_pass<N, 1>(sm, cnt, p.S); __syncthreads(); }
    if (p.d >= 4) { tile_pass<N, N2>(sm, cnt, p.S); __syncthreads(); }
    if (p.d >= 6) { tile_pass<N, N4>(sm, cnt, p.S); __syncthreads(); }
    if (p.d == 1) { line_pass<N, 1>(sm, cnt, p.S); __syncthreads(); }
    if (p.d == 3) { line_pass<N, N2>(sm, cnt, p.S); __syncthreads(); }
    if (p.d == 5) { line_pass<N, N4>(sm, cnt, p.S); __syncthreads(); }
    double *dst = p.v + b * (long long)full;
    // consecutive threads read consecutive (conflict-free) padded slots and write one contiguous segment per warp
    if constexpr (N % 2 == 0) {
      for (int e = 2 * threadIdx.x; e < cnt; e += 2 * blockDim.x)
        __stcs(reinterpret_cast<double2 *>(dst + e), *reinterpret_cast<const double2 *>(&sm[padded<N>(e)]));
    } else {
      for (int e = threadIdx.x; e < cnt; e += blockDim.x) __stcs(dst + e, sm[padded<N>(e)]);
    }
    __syncthreads();  // the buffer has been read out before it is refilled
    if (p.nbuf == 2) {
      cur ^= 1;
    } else {
      if (nxt < nb) issue(nxt, smem);
      cp_async_commit();
    }
  }
  cp_async_wait<0>();
}

constexpr int kBatchDoubles = 4096;
constexpr size_t kMaxSmem = 200 * 1024;

long long ipow_ll(int b, int e) {
  long long r = 1;
  for (int i = 0; i < e; ++i) r *= b;
  return r;
}

// bytes of one staging buffer (the kernel's bufsz)
size_t smem_of(long long doubles, int n) {
  return (size_t)(n % 2 == 0 ? doubles + 2 * (doubles >> 4) + 2 : doubles + (doubles >> 5) + 1) * sizeof(double);
}

template <int N>
cudaError_t launch_n(BasisParams &p, cudaStream_t s, int sms) {
  const long long ND = ipow_ll(N, p.d);
  long long cb = kBatchDoubles / ND;
  if (cb < 1) cb = 1;
  if (cb > p.ncells) cb = p.ncells;
  p.cb = (int)cb;
  const size_t one = smem_of(cb * ND, N);
  p.nbuf = 2 * one <= kMaxSmem ? 2 : 1;
  const size_t smem = p.nbuf * one;
  cudaError_t e = cudaFuncSetAttribute(basis_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxSmem);
  if (e != cudaSuccess) return e;
  const long long nb = (p.ncells + cb - 1) / cb;
  int per_sm = (int)((227 * 1024) / (smem + 1024));
  const int by_regs = N <= 3 ? 4 : N == 4 ? 3 : N == 5 ? 2 : 1;  // the kernel's launch bounds
  if (per_sm > by_regs) per_sm = by_regs;
  if (per_sm < 1) per_sm = 1;
  const long long cap = (long long)sms * per_sm;
  basis_kernel<N><<<(unsigned)(nb < cap ? nb : cap), 256, smem, s>>>(p);
  return cudaGetLastError();
}

}  // namespace

bool basis_kernel_supported(int d, int n) {
  return d >= 1 && d <= 6 && n >= 2 && n <= kMaxN && smem_of(ipow_ll(n, d), n) <= kMaxSmem;
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
