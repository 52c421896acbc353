// hd_fcl.cu -- the face-centric loop (FCL) comparison path of v <- A(u).
//
// The paper evaluates the DG operator either element-centric (ECL: each cell with its 2d faces, every flux
// computed twice; the product path, hd_cell.cuh) or face-centric (FCL: a cell loop for the volume
// integrals plus a face loop that computes the numerical flux of every face ONCE and tests it on both
// sides), and benchmarks the two against each other (Figure fig:performance:
// alternatives:fcl). On the GPU the face loop's "test on both sides" writes the same cell from two faces,
// so the loop is split into three race-free passes (DESIGN.md §6 "FCL"):
//
//   fcl_cell_kernel   per cell (one CTA, cell staged in smem): v <- volume term of Alg. 2 step 2-4 (weak
//                     form, Gauss collocation), and both face traces u(xi_i = 0), u(xi_i = 1) of every dim
//                     (Alg. 2 steps 1-2 on the faces) -> trace buffer T[i][side][cell][face point]
//   fcl_face_kernel   per face (cell L, dim i, face point): F = numerical flux of
//                     (u- = T[i][1][L], u+ = T[i][0][R], a_i n), times the face quadrature weight |J|/h_i w_f
//                     -> G[i][L][face point]: the flux of face (L, R) computed once
//   fcl_lift_kernel   per DoF: v_m -= sum_i l_{m_i}(1) G[i][cell] - l_{m_i}(0) G[i][left_i(cell)]
//                     (Alg. 2 step 4 for both sides of every face; F_R = -F_L by conservation)
//
// Plain CUDA (no schedule, no trace protocol): the point is the loop structure the paper compares, with the
// same arithmetic as the product operator up to rounding order. Single-rank meshes; any flux sign pattern.
#include <cuda_runtime.h>

#include "hd_internal.h"

namespace hd {

namespace {

constexpr __host__ __device__ int fpow(int b, int e) { return e == 0 ? 1 : b * fpow(b, e - 1); }

template <int D, int N>
__global__ void __launch_bounds__(256) fcl_cell_kernel(const __grid_constant__ FclParams p) {
  constexpr int ND = fpow(N, D), FN = ND / N;
  extern __shared__ double su[];
  for (long long cell = blockIdx.x; cell < p.ncells; cell += gridDim.x) {
    __syncthreads();
    const double *uc = p.u + cell * ND;
    if constexpr (ND % 2 == 0) {
      for (int e = threadIdx.x; e < ND / 2; e += blockDim.x)
        reinterpret_cast<double2 *>(su)[e] = __ldcs(reinterpret_cast<const double2 *>(uc) + e);
    } else {
      for (int e = threadIdx.x; e < ND; e += blockDim.x) su[e] = __ldcs(uc + e);
    }
    long long cc[D];
    {
      long long r = cell;
#pragma unroll
      for (int j = 0; j < D; ++j) {
        cc[j] = r % p.L[j];
        r /= p.L[j];
      }
    }
    __syncthreads();
    // volume term: b_m = sum_i |J|/h_i prod_{j != i} w_{m_j} a_i(z_m) sum_q w_q l'_{m_i}(xi_q) u_(m, m_i -> q)
    for (int m = threadIdx.x; m < ND; m += blockDim.x) {
      int mi[D];
      {
        int r = m;
#pragma unroll
        for (int j = 0; j < D; ++j) {
          mi[j] = r % N;
          r /= N;
        }
      }
      double b = 0.0;
#pragma unroll
      for (int i = 0; i < D; ++i) {
        double a = p.a_const[i], wf = 1.0;
#pragma unroll
        for (int j = 0; j < D; ++j) {
          if (j == i) continue;
          a += p.a_lin[i][j] * (p.lo[j] + ((double)cc[j] + p.xi[mi[j]]) * p.h[j]);
          wf *= p.w[mi[j]];
        }
        // Vlasov-Poisson: a_{d_x + l} = ... - E_l(x) at the DoF's x node (P:3963 a = (v, -E(x)))
        if (p.E && i >= p.d_x) a -= p.E[((long long)(i - p.d_x) * p.ncx + cell % p.ncx) * p.nx + m % p.nx];
        int stride = 1;
        for (int j = 0; j < i; ++j) stride *= N;
        const int base = m - mi[i] * stride;
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < N; ++q) s += p.Dw[mi[i]][q] * su[base + q * stride];
        b += p.jdet_h[i] * wf * a * s;
      }
      __stcs(p.v + cell * ND + m, b);
    }
    // face traces of every dim: T[i][s][cell][f] = sum_j l_j(s) u_(f, m_i = j)
    for (int e = threadIdx.x; e < D * FN; e += blockDim.x) {
      const int i = e / FN, f = e - i * FN;
      int stride = 1;
      for (int j = 0; j < i; ++j) stride *= N;
      const int base = (f % stride) + (f / stride) * stride * N;
      double t0 = 0.0, t1 = 0.0;
#pragma unroll
      for (int j = 0; j < N; ++j) {
        t0 += p.l0[j] * su[base + j * stride];
        t1 += p.l1[j] * su[base + j * stride];
      }
      p.tr[((long long)(2 * i) * p.ncells + cell) * FN + f] = t0;
      p.tr[((long long)(2 * i + 1) * p.ncells + cell) * FN + f] = t1;
    }
  }
}

template <int D, int N>
__global__ void __launch_bounds__(256) fcl_face_kernel(const __grid_constant__ FclParams p) {
  constexpr int ND = fpow(N, D), FN = ND / N;
  const long long total = (long long)D * p.ncells * FN;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int f = (int)(e % FN);  // FN: compile-time divisor
    const long long r0 = e / FN;
    const int i = (int)(r0 / p.ncells);
    const unsigned cell = (unsigned)(r0 - (long long)i * p.ncells);  // < 2^31 cells (hd_create_mesh)
    unsigned cc[D], ci = 0, csi = 1;
    {
      unsigned r = cell, s = 1;
#pragma unroll
      for (int j = 0; j < D; ++j) {
        const unsigned q = r / p.L32[j];
        cc[j] = r - q * p.L32[j];
        r = q;
        if (j == i) {
          ci = cc[j];
          csi = s;
        }
        s *= p.L32[j];
      }
    }
    // node indices of the face point (the dims j != i in order, fastest first)
    double a = p.a_const[i], wf = 1.0;
    {
      int r = f;
#pragma unroll
      for (int j = 0; j < D; ++j) {
        if (j == i) continue;
        const int mj = r % N;
        r /= N;
        a += p.a_lin[i][j] * (p.lo[j] + ((double)cc[j] + p.xi[mj]) * p.h[j]);
        wf *= p.w[mj];
      }
    }
    if (p.E && i >= p.d_x) a -= p.E[((long long)(i - p.d_x) * p.ncx + cell % p.ncx) * p.nx + f % p.nx];
    const unsigned right = ci + 1 < p.L32[i] ? cell + csi : cell - (p.L32[i] - 1) * csi;  // periodic
    const double um = p.tr[((long long)(2 * i + 1) * p.ncells + cell) * FN + f];
    const double up = p.tr[((long long)(2 * i) * p.ncells + right) * FN + f];
    // central a.n (u- + u+)/2; upwind adds |a.n| (u- - u+)/2 (n = +e_i seen from L)
    double F = a * 0.5 * (um + up);
    if (p.flux == 0) F += fabs(a) * 0.5 * (um - up);
    p.G[((long long)i * p.ncells + cell) * FN + f] = F * wf * p.jdet_h[i];
  }
}

template <int D, int N>
__global__ void __launch_bounds__(256) fcl_lift_kernel(const __grid_constant__ FclParams p) {
  constexpr int ND = fpow(N, D), FN = ND / N;
  const long long total = p.ncells * ND;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const unsigned cell = (unsigned)(e / ND);  // ND: compile-time divisor; < 2^31 cells
    const int m = (int)(e - (long long)cell * ND);
    unsigned cc[D], cs[D];
    {
      unsigned r = cell, s = 1;
#pragma unroll
      for (int j = 0; j < D; ++j) {
        const unsigned q = r / p.L32[j];
        cc[j] = r - q * p.L32[j];
        r = q;
        cs[j] = s;
        s *= p.L32[j];
      }
    }
    double acc = 0.0;
    int stride = 1;
#pragma unroll
    for (int i = 0; i < D; ++i) {
      const int mi = (m / stride) % N;
      const int f = (m % stride) + (m / (stride * N)) * stride;
      const unsigned left = cc[i] > 0 ? cell - cs[i] : cell + (p.L32[i] - 1) * cs[i];  // periodic
      const double gr = __ldg(p.G + ((long long)i * p.ncells + cell) * FN + f);   // own right face, n = +e_i
      const double gl = __ldg(p.G + ((long long)i * p.ncells + left) * FN + f);   // own left face: -F of L
      acc += p.l1[mi] * gr - p.l0[mi] * gl;
      stride *= N;
    }
    p.v[e] -= acc;
  }
}

template <int D, int N>
cudaError_t launch_fcl_dn(const FclParams &p, cudaStream_t s, int sms) {
  constexpr int ND = fpow(N, D);
  const size_t smem = (size_t)ND * sizeof(double);
  if (smem > 200 * 1024) return cudaErrorNotSupported;
  cudaError_t e = cudaFuncSetAttribute(fcl_cell_kernel<D, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  long long g1 = p.ncells < (long long)sms * 8 ? p.ncells : (long long)sms * 8;
  if (g1 < 1) return cudaSuccess;
  fcl_cell_kernel<D, N><<<(unsigned)g1, 256, smem, s>>>(p);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const long long nf = (long long)D * p.ncells * (ND / N), nv = p.ncells * ND;
  long long g2 = (nf + 255) / 256, g3 = (nv + 255) / 256;
  const long long cap = (long long)sms * 16;
  fcl_face_kernel<D, N><<<(unsigned)(g2 < cap ? g2 : cap), 256, 0, s>>>(p);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  fcl_lift_kernel<D, N><<<(unsigned)(g3 < cap ? g3 : cap), 256, 0, s>>>(p);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// Vlasov-Poisson (Eq. equ:vp:close; DESIGN.md §6 "Vlasov-Poisson").
// rho(x) = 1 - int f dv at every x node: one CTA per x cell; thread e of the cell-local index sums
// its value over the v cells (coalesced: consecutive threads, consecutive DoFs), then the x nodes sum their
// v nodes from shared memory. Fixed summation order (deterministic).
__global__ void __launch_bounds__(256) vp_density_kernel(const __grid_constant__ VpParams p, const double *f,
                                                         double *rho) {
  extern __shared__ double S[];  // [ND]
  for (long long cx = blockIdx.x; cx < p.ncx; cx += gridDim.x) {
    __syncthreads();
    for (int e = threadIdx.x; e < p.ND; e += blockDim.x) {
      const double *fc = f + cx * p.ND + e;
      double s = 0.0;
      for (long long cv = 0; cv < p.ncv; ++cv) s += __ldcs(fc + cv * p.ncx * p.ND);
      S[e] = p.wv[e / p.nx] * s;
    }
    __syncthreads();
    for (int jx = threadIdx.x; jx < p.nx; jx += blockDim.x) {
      double s = 0.0;
      for (int jv = 0; jv < p.nv; ++jv) s += S[jx + jv * p.nx];
      rho[cx * p.nx + jx] = 1.0 - s;
    }
  }
}

// x-node coordinates of (x cell cx, x node jx)
__device__ __forceinline__ void vp_xnode(const VpParams &p, long long cx, int jx, double *x, double *w) {
  double ww = 1.0;
  for (int i = 0; i < p.d_x; ++i) {
    const long long c = cx % p.Lx[i];
    cx /= p.Lx[i];
    const int j = jx % p.n;
    jx /= p.n;
    x[i] = p.lo[i] + ((double)c + p.xi[j]) * p.h[i];
    ww *= p.w[j] * p.h[i];
  }
  *w = ww;
}

// Fourier coefficients of rho_h by its Gauss rule: rhohat(m) = |Omega_x|^-1 sum_nodes W rho e^{-i k.x},
// k_i = 2 pi m_i / L_i, |m_i| <= K_i: one CTA per mode, threads over the x nodes, fixed-shape tree reduction
// in shared memory (deterministic).
__global__ void __launch_bounds__(256) vp_rhohat_kernel(const __grid_constant__ VpParams p, const double *rho,
                                                        double *rhohat) {
  __shared__ double sre[256], sim[256];
  for (long long q = blockIdx.x; q < p.nmodes; q += gridDim.x) {
    double k[3] = {0, 0, 0};
    long long r = q;
    for (int i = 0; i < p.d_x; ++i) {
      const long long w = 2 * p.K[i] + 1;
      k[i] = 2.0 * M_PI * (double)(r % w - p.K[i]) / p.Lbox[i];
      r /= w;
    }
    double re = 0.0, im = 0.0;
    const long long nxn = p.ncx * p.nx;
    for (long long e = threadIdx.x; e < nxn; e += blockDim.x) {
      const long long cx = e / p.nx;
      double x[3], W;
      vp_xnode(p, cx, (int)(e - cx * p.nx), x, &W);
      double ph = 0.0;
      for (int i = 0; i < p.d_x; ++i) ph += k[i] * x[i];
      double sn, cs;
      sincos(ph, &sn, &cs);
      const double t = W * rho[e];
      re += t * cs;
      im -= t * sn;
    }
    __syncthreads();
    sre[threadIdx.x] = re;
    sim[threadIdx.x] = im;
    __syncthreads();
    for (int h = 128; h > 0; h >>= 1) {
      if (threadIdx.x < h) {
        sre[threadIdx.x] += sre[threadIdx.x + h];
        sim[threadIdx.x] += sim[threadIdx.x + h];
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      rhohat[2 * q] = sre[0] / p.vol_x;
      rhohat[2 * q + 1] = sim[0] / p.vol_x;
    }
  }
}

// E = -grad phi, -lap phi = rho: E_i(x) = sum_{m != 0} k_i / |k|^2 (Re rhohat sin(k.x) + Im rhohat cos(k.x)),
// at every x node: thread per (x cell, x node); out E[i][cx][jx].
__global__ void __launch_bounds__(256) vp_efield_kernel(const __grid_constant__ VpParams p, const double *rhohat,
                                                        double *E) {
  const long long nxn = p.ncx * p.nx;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nxn; e += (long long)gridDim.x * blockDim.x) {
    const long long cx = e / p.nx;
    double x[3], W;
    vp_xnode(p, cx, (int)(e - cx * p.nx), x, &W);
    double acc[3] = {0, 0, 0};
    for (long long q = 0; q < p.nmodes; ++q) {
      double k[3] = {0, 0, 0}, k2 = 0.0;
      long long r = q;
      for (int i = 0; i < p.d_x; ++i) {
        const long long w = 2 * p.K[i] + 1;
        k[i] = 2.0 * M_PI * (double)(r % w - p.K[i]) / p.Lbox[i];
        k2 += k[i] * k[i];
        r /= w;
      }
      if (k2 == 0.0) continue;
      double ph = 0.0;
      for (int i = 0; i < p.d_x; ++i) ph += k[i] * x[i];
      double sn, cs;
      sincos(ph, &sn, &cs);
      const double g = rhohat[2 * q] * sn + rhohat[2 * q + 1] * cs;
      for (int i = 0; i < p.d_x; ++i) acc[i] += k[i] / k2 * g;
    }
    for (int i = 0; i < p.d_x; ++i) E[(long long)i * nxn + e] = acc[i];
  }
}

// 2N low-storage update of one stage: dU <- A_s dU + dt w (first stage: dU <- dt w); U <- U + B_s dU
__global__ void __launch_bounds__(256) vp_update_kernel(double *U, double *dU, const double *w, long long n, double A,
                                                        double B, double dt, int first) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const double d = first ? dt * w[e] : A * dU[e] + dt * w[e];
    dU[e] = d;
    U[e] = U[e] + B * d;
  }
}

}  // namespace

cudaError_t launch_vp_fields(const VpParams &p, const double *f, double *rho, double *rhohat, double *E, cudaStream_t s,
                             long long *launches, int sms) {
  const long long nxn = p.ncx * p.nx;
  const long long cap = (long long)sms * 16;
  auto grid = [&](long long n) { long long g = (n + 255) / 256; return (unsigned)(g < 1 ? 1 : (g < cap ? g : cap)); };
  const size_t smem = (size_t)p.ND * sizeof(double);
  cudaError_t e = cudaFuncSetAttribute(vp_density_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  vp_density_kernel<<<(unsigned)(p.ncx < cap ? p.ncx : cap), 256, smem, s>>>(p, f, rho);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  vp_rhohat_kernel<<<(unsigned)(p.nmodes < cap ? p.nmodes : cap), 256, 0, s>>>(p, rho, rhohat);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  vp_efield_kernel<<<grid(nxn), 256, 0, s>>>(p, rhohat, E);
  if (launches) *launches += 3;
  return cudaGetLastError();
}

cudaError_t launch_vp_update(double *U, double *dU, const double *w, long long n, double A, double B, double dt,
                             int first, cudaStream_t s, long long *launches, int sms) {
  long long g = (n + 255) / 256;
  const long long cap = (long long)sms * 16;
  if (g > cap) g = cap;
  if (g < 1) return cudaSuccess;
  vp_update_kernel<<<(unsigned)g, 256, 0, s>>>(U, dU, w, n, A, B, dt, first);
  if (launches) *launches += 1;
  return cudaGetLastError();
}

bool fcl_supported(int d, int n) {
  if (d < 2 || d > 6 || n < 2 || n > 6) return false;
  long long nd = 1;
  for (int i = 0; i < d; ++i) nd *= n;
  return nd * (long long)sizeof(double) <= 200 * 1024;
}

cudaError_t launch_fcl(int d, int n, const FclParams &p, cudaStream_t s, long long *launches, int sms) {
  if (!fcl_supported(d, n)) return cudaErrorNotSupported;
  if (launches) *launches += 3;
#define HD_FCL_N(D)                                          \
  switch (n) {                                               \
    case 2: return launch_fcl_dn<D, 2>(p, s, sms);           \
    case 3: return launch_fcl_dn<D, 3>(p, s, sms);           \
    case 4: return launch_fcl_dn<D, 4>(p, s, sms);           \
    case 5: return launch_fcl_dn<D, 5>(p, s, sms);           \
    case 6: if constexpr (fpow(6, D) * 8 <= 200 * 1024) return launch_fcl_dn<D, 6>(p, s, sms); else break; \
    default: break;                                          \
  }                                                          \
  break;
  switch (d) {
    case 2: HD_FCL_N(2)
    case 3: HD_FCL_N(3)
    case 4: HD_FCL_N(4)
    case 5: HD_FCL_N(5)
    case 6: HD_FCL_N(6)
    default: break;
  }
#undef HD_FCL_N
  return cudaErrorNotSupported;
}

}  // namespace hd
