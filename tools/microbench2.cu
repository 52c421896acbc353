// Design microbenchmarks, round 2 (not part of the product path):
//  1. DFMA dependent-chain latency (one warp, one chain).
//  2. DFMA alone vs DMMA alone vs both interleaved in the same warps: do the FP64 pipe and the f64
//     mma path run concurrently?
//  3. smem LDS.64 / LDS.128 bandwidth with conflict-free addresses.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb2 microbench2.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__global__ void lat_kernel(double *out, int iters, double a, double b, long long *cyc) {
  double x = threadIdx.x * 1e-3;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) x = fma(x, a, b);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = t1 - t0;
  if (x == 12345.678) out[0] = x;
}

template <int CH, int MM>
__global__ void mix_kernel(double *out, int iters, double a, double b) {
  double x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-3 + c;
  double ma = threadIdx.x * 1e-3, mb = 1.0001;
  double acc[MM > 0 ? MM : 1][2];
#pragma unroll
  for (int k = 0; k < (MM > 0 ? MM : 1); ++k) { acc[k][0] = k; acc[k][1] = -k; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = fma(x[c], a, b);
#pragma unroll
    for (int k = 0; k < MM; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[k][0]), "+d"(acc[k][1]) : "d"(ma), "d"(mb));
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
#pragma unroll
  for (int k = 0; k < (MM > 0 ? MM : 1); ++k) s += acc[k][0] + acc[k][1];
  if (s == 12345.678) out[0] = s;
}

template <int W>
__global__ void lds_kernel(double *out, int iters) {
  extern __shared__ double sm[];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = i;
  __syncthreads();
  double s = 0;
  const int base = (threadIdx.x * W) & 4095;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      if constexpr (W == 1) s += sm[(base + k * 256 + i) & 8191];
      else {
        double2 v = *reinterpret_cast<const double2 *>(sm + ((base + k * 512 + 2 * i) & 8190));
        s += v.x + v.y;
      }
    }
  }
  if (s == 12345.678) out[0] = s;
}

int main() {
  cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr, 0));
  const int sms = pr.multiProcessorCount;
  double *dout; CK(cudaMalloc(&dout, 64));
  long long *dcyc; CK(cudaMalloc(&dcyc, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  {
    lat_kernel<<<1, 32>>>(dout, 10, 1.0000001, 1e-9, dcyc);
    lat_kernel<<<1, 32>>>(dout, 1000, 1.0000001, 1e-9, dcyc);
    CK(cudaDeviceSynchronize());
    long long c; CK(cudaMemcpy(&c, dcyc, 8, cudaMemcpyDeviceToHost));
    printf("{\"test\":\"dfma_latency\",\"cycles_per_dep_fma\":%.2f}\n", c / 16000.0);
  }
  auto run = [&](const char *name, void (*k)(double *, int, double, double), int iters, double fma_per_iter_thread,
                 double mma_per_iter_warp, int threads, int bpsm) {
    int blocks = sms * bpsm;
    k<<<blocks, threads>>>(dout, 10, 1.0000001, 1e-9);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      k<<<blocks, threads>>>(dout, iters, 1.0000001, 1e-9);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double dfma = (double)blocks * threads * iters * fma_per_iter_thread;
    double mfma = (double)blocks * (threads / 32) * iters * mma_per_iter_warp * 256;
    printf("{\"test\":\"%s\",\"threads\":%d,\"blocks_per_sm\":%d,\"ms\":%.3f,\"dfma_tfma\":%.3f,\"dmma_tfma\":%.3f,\"total_tfma\":%.3f}\n",
           name, threads, bpsm, best, dfma / best / 1e9, mfma / best / 1e9, (dfma + mfma) / best / 1e9);
  };
  for (int bpsm : {1, 2, 4, 8}) {
    run("dfma8", mix_kernel<8, 0>, 4000, 8, 0, 256, bpsm);
    run("dmma4", mix_kernel<1, 4>, 2000, 1, 4, 256, bpsm);
    run("dfma8+dmma1", mix_kernel<8, 1>, 4000, 8, 1, 256, bpsm);
    run("dfma8+dmma2", mix_kernel<8, 2>, 4000, 8, 2, 256, bpsm);
    run("dfma4+dmma2", mix_kernel<4, 2>, 4000, 4, 2, 256, bpsm);
  }
  {
    CK(cudaFuncSetAttribute(lds_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
    CK(cudaFuncSetAttribute(lds_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
    for (int w : {1, 2}) {
      int blocks = sms * 2, threads = 512, iters = 4000;
      float best = 1e30f;
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        if (w == 1) lds_kernel<1><<<blocks, threads, 65536>>>(dout, iters);
        else lds_kernel<2><<<blocks, threads, 65536>>>(dout, iters);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      }
      double bytes = (double)blocks * threads * iters * 16 * 8 * w;
      printf("{\"test\":\"lds%d\",\"bytes_per_clk_per_sm_at_1965\":%.1f}\n", 64 * w,
             bytes / (best * 1e-3) / sms / 1.965e9);
    }
  }
  return 0;
}
