// Hardware microbenchmarks for design decisions (not part of the product path).
// FP64 FMA rate, f64 mma.sync rate, L2 re-read bandwidth vs working-set size,
// HBM copy bandwidth. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb microbench.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

template <int CHAINS>
__global__ void dfma_kernel(double *out, int iters, double a, double b) {
  double x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_kernel(double *out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0001;
  double c[4][2];
#pragma unroll
  for (int k = 0; k < 4; ++k) { c[k][0] = k; c[k][1] = -k; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void read_kernel(const double2 *__restrict__ p, size_t n2, int reps, double *out) {
  double acc = 0;
  size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x, stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (size_t i = tid; i < n2; i += stride) { double2 v = p[i]; acc += v.x + v.y; }
  if (acc == 12345.678) out[0] = acc;
}

__global__ void copy_kernel(const double2 *__restrict__ a, double2 *__restrict__ b, size_t n2) {
  size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x, stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = tid; i < n2; i += stride) b[i] = a[i];
}

int main() {
  cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr, 0));
  int l2 = 0, smemopt = 0, clk = 0, memclk = 0;
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
  cudaDeviceGetAttribute(&smemopt, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaDeviceGetAttribute(&memclk, cudaDevAttrMemoryClockRate, 0);
  size_t fr, tot; CK(cudaMemGetInfo(&fr, &tot));
  printf("{\"name\":\"%s\",\"sms\":%d,\"l2_bytes\":%d,\"smem_optin\":%d,\"clock_khz\":%d,\"memclk_khz\":%d,\"mem_free\":%zu,\"mem_total\":%zu,\"persisting_l2_max\":%d}\n",
         pr.name, pr.multiProcessorCount, l2, smemopt, clk, memclk, fr, tot, pr.persistingL2CacheMaxSize);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  double *dout; CK(cudaMalloc(&dout, 64));
  int sms = pr.multiProcessorCount;
  // DFMA
  {
    int iters = 20000, blocks = sms * 8, threads = 256;
    dfma_kernel<8><<<blocks, threads>>>(dout, 100, 1.0000001, 1e-9);
    CK(cudaDeviceSynchronize());
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      dfma_kernel<8><<<blocks, threads>>>(dout, iters, 1.0000001, 1e-9);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double fmas = (double)blocks * threads * iters * 8;
      printf("{\"test\":\"dfma\",\"ms\":%.3f,\"tfma_per_s\":%.3f,\"fma_per_clk_per_sm_at_1965\":%.2f}\n", ms, fmas / ms / 1e9,
             fmas / (ms * 1e-3) / sms / 1.965e9);
    }
  }
  // DMMA m8n8k4: 8*8*4 = 256 FMA per warp-instruction
  {
    int iters = 5000, blocks = sms * 8, threads = 256;
    dmma_kernel<<<blocks, threads>>>(dout, 10);
    CK(cudaDeviceSynchronize());
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      dmma_kernel<<<blocks, threads>>>(dout, iters);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double fmas = (double)blocks * (threads / 32) * iters * 4 * 256;
      printf("{\"test\":\"dmma_m8n8k4\",\"ms\":%.3f,\"tfma_per_s\":%.3f}\n", ms, fmas / ms / 1e9);
    }
  }
  // L2 read bandwidth vs working set
  {
    size_t maxb = (size_t)1 << 30;
    double2 *buf; CK(cudaMalloc(&buf, maxb)); CK(cudaMemset(buf, 0, maxb));
    size_t sizes[] = {(size_t)8 << 20, (size_t)16 << 20, (size_t)32 << 20, (size_t)48 << 20, (size_t)64 << 20,
                      (size_t)80 << 20, (size_t)96 << 20, (size_t)112 << 20, (size_t)128 << 20, (size_t)1 << 30};
    for (size_t sz : sizes) {
      size_t n2 = sz / 16;
      int reps = (int)((size_t)(4ull << 30) / sz); if (reps < 2) reps = 2;
      int blocks = sms * 8, threads = 512;
      read_kernel<<<blocks, threads>>>(buf, n2, 1, dout);
      CK(cudaDeviceSynchronize());
      float best = 1e30f;
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        read_kernel<<<blocks, threads>>>(buf, n2, reps, dout);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      }
      printf("{\"test\":\"read\",\"mb\":%zu,\"gbs\":%.1f}\n", sz >> 20, (double)sz * reps / best / 1e6);
    }
    CK(cudaFree(buf));
  }
  // HBM copy
  {
    size_t sz = (size_t)4 << 30;
    double2 *a, *b; CK(cudaMalloc(&a, sz)); CK(cudaMalloc(&b, sz));
    CK(cudaMemset(a, 0, sz)); CK(cudaMemset(b, 0, sz));
    size_t n2 = sz / 16;
    for (int bl : {sms * 4, sms * 8, sms * 16}) {
      copy_kernel<<<bl, 512>>>(a, b, n2); CK(cudaDeviceSynchronize());
      float best = 1e30f;
      for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0); copy_kernel<<<bl, 512>>>(a, b, n2); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      }
      printf("{\"test\":\"copy\",\"blocks\":%d,\"gbs\":%.1f}\n", bl, 2.0 * sz / best / 1e6);
    }
  }
  return 0;
}
