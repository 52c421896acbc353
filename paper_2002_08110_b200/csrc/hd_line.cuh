// hd_line.cuh -- the "line" variant of the fused cell kernel: the same operator, units,
// trace protocol and RK epilogue as hd_cell.cuh, but the cell is swept ONE DIM PER PASS with one 1D line
// per thread iteration and the running accumulator in shared memory. Per thread only one line (n values)
// is live, so a thread needs few registers and three CTAs fit on an SM: the barriers of one CTA and the
// cell loads (not prefetched: single buffer) are hidden by the others instead of inside the CTA.
// Face (trace) layout: face point f of dim X = the line index, i.e. the cell-local digits of the dims
// other than X in ascending order (line_base).
#pragma once
#ifndef HD_LINE_MINB
#define HD_LINE_MINB 3
#endif

namespace hd {

// cell-local offset (dim-X digit 0) of line f of dim X
template <int D, int N, int X>
__host__ __device__ __forceinline__ int line_base(int f) {
  int off = 0, m = 1;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    if (j != X) {
      off += (f % N) * m;
      f /= N;
    }
    m *= N;
  }
  return off;
}
template <int D, int N>
__device__ __forceinline__ int line_base_rt(int X, int f) {
  int off = 0, m = 1;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    if (j != X) {
      off += (f % N) * m;
      f /= N;
    }
    m *= N;
  }
  return off;
}

// One pass over dim X for every line of the group. FIRSTP: the accumulator is written, not read;
// LASTP: the epilogue (weak-form scaling or LSRK update) replaces the write-back.
template <int D, int N, int MODE, int X>
__device__ __forceinline__ void line_pass(const CellParams &p, const CellInfo *info, const double *stab, const double *U,
                                          double *ACC, double *carry, int tid, int nthreads) {
  using G = CGeo<D, N>;
  constexpr int SX = ipow(N, X);
  constexpr bool FIRSTP = X == 0, LASTP = X == D - 1;
  const Tables1D &T = c_tab[N];
  const int CT = p.CT;
  const double facX = p.dtfac * p.inv_h[X];
  for (int L = tid; L < CT * G::FN; L += nthreads) {
    const int k = L / G::FN, f = L - k * G::FN;
    const CellInfo &ci = info[k];
    const int b = line_base<D, N, X>(f);
    const double *Uk = U + (size_t)k * G::ND + b;
    double *Ak = ACC + (size_t)k * G::ND + b;
    double u[N];
    if constexpr (X == 0 && N % 2 == 0) {
#pragma unroll
      for (int j = 0; j < N; j += 2) {
        const double2 v2 = *reinterpret_cast<const double2 *>(Uk + j);
        u[j] = v2.x;
        u[j + 1] = v2.y;
      }
    } else {
#pragma unroll
      for (int j = 0; j < N; ++j) u[j] = Uk[j * SX];
    }
    const int sg = ci.sg[X];
    const unsigned char src = ci.src[X], out = ci.out[X];
    // upwind trace value of this line's face point (issued before the contraction)
    double t = 0.0;
    if (src == kSrcPub || src == kSrcHalo) t = __ldcg(ci.tsrc[X] + f);
    else if (src == kSrcCarry) t = carry[(size_t)k * G::FN + f];
    // line speed: a_X at the line (a_X does not depend on z_X)
    double w = ci.base[X];
    {
      int ff = f;
#pragma unroll
      for (int j = 0; j < D; ++j) {
        if (j == X) continue;
        const int m = ff % N;
        ff /= N;
        if (p.a_lin[X][j] != 0.0) w = fma(p.a_lin[X][j] * p.h[j], stab[m], w);
      }
    }
    const double s = w * facX;
    // own downwind trace (publish / carry) and the volume + own-face term
    if (out != kOutNone) {
      double tr = T.tau[sg][0] * u[0];
#pragma unroll
      for (int j = 1; j < N; ++j) tr = fma(T.tau[sg][j], u[j], tr);
      if (out == kOutCarry) carry[(size_t)k * G::FN + f] = tr;
      else __stcg(p.tbuf[X] + ((size_t)ci.unit * p.UC + ci.cu) * G::FN + f, tr);
    }
    double y[N];
#pragma unroll
    for (int a = 0; a < N; ++a) y[a] = T.K[sg][a][0] * u[0];
#pragma unroll
    for (int j = 1; j < N; ++j)
#pragma unroll
      for (int a = 0; a < N; ++a) y[a] = fma(T.K[sg][a][j], u[j], y[a]);
    // the upwind trace from the group (smem) or the neighbour cell (global)
    if (src == kSrcGroup) {
      const double *nb = U + (size_t)ci.nb[X] * G::ND + b;
      t = T.tau[sg][0] * nb[0];
#pragma unroll
      for (int j = 1; j < N; ++j) t = fma(T.tau[sg][j], nb[j * SX], t);
    } else if (src == kSrcDirect) {
      const double *nb = p.u + (size_t)ci.nb[X] * G::ND + b;
      double v[N];
#pragma unroll
      for (int j = 0; j < N; ++j) v[j] = __ldg(nb + j * SX);
      t = T.tau[sg][0] * v[0];
#pragma unroll
      for (int j = 1; j < N; ++j) t = fma(T.tau[sg][j], v[j], t);
    }
    // rank-1 lift and speed: contribution of dim X to (M^-1 A u) along the line
    {
      const double st = s * t;
#pragma unroll
      for (int a = 0; a < N; ++a) y[a] = fma(T.lam[sg][a], st, s * y[a]);
    }
    // y: contribution of dim X (volume, own face, rank-1 lift of the upwind trace) to (M^-1 A u)
    if constexpr (!LASTP) {
      if constexpr (FIRSTP && N % 2 == 0) {
#pragma unroll
        for (int a = 0; a < N; a += 2) *reinterpret_cast<double2 *>(Ak + a) = make_double2(y[a], y[a + 1]);
      } else {
#pragma unroll
        for (int a = 0; a < N; ++a) {
          if constexpr (FIRSTP) Ak[a * SX] = y[a];
          else Ak[a * SX] += y[a];
        }
      }
    } else {
      const size_t g0 = (size_t)ci.cell * G::ND + b;
      if constexpr (MODE == kModeAdvection) {
        // weak form: v = M (M^-1 A u), M_qq = |J| prod_i w_{q_i}
        double wr = p.jdet;
        {
          int ff = f;
#pragma unroll
          for (int j = 0; j < D; ++j) {
            if (j == X) continue;
            wr *= stab[8 + ff % N];
            ff /= N;
          }
        }
#pragma unroll
        for (int a = 0; a < N; ++a) {
          const double acc = FIRSTP ? y[a] : Ak[a * SX] + y[a];
          __stcs(p.out + g0 + a * SX, acc * (wr * T.w[a]));
        }
      } else {
        // LSRK 2N stage: dU <- A_s dU + dt M^-1 A(U); U_new <- U + B_s dU
        double du[N];
        if constexpr (MODE == kModeRK) {
#pragma unroll
          for (int a = 0; a < N; ++a) du[a] = __ldcs(p.du + g0 + a * SX);
        }
#pragma unroll
        for (int a = 0; a < N; ++a) {
          double dun = FIRSTP ? y[a] : Ak[a * SX] + y[a];
          if constexpr (MODE == kModeRK) dun = fma(p.rk_a, du[a], dun);
          __stcs(p.du + g0 + a * SX, dun);
          __stcs(p.out + g0 + a * SX, fma(p.rk_b, dun, u[a]));
        }
      }
    }
    // a published trace is consumed exactly once: drop its L2 line (16 face points of consecutive lanes
    // of this warp, all of the same cell) without write-back once the warp has read it
    if constexpr (G::FN % 32 == 0) {
      if (p.discard && p.pubany) {
        __syncwarp();
        if (src == kSrcPub && (f & 15) == 0) discard_l2_line(ci.tsrc[X] + f);
      }
    }
  }
}

template <int D, int N>
__host__ __device__ constexpr int line_smem_bytes(int CT) {
  using G = CGeo<D, N>;
  return (2 * CT * G::ND + CT * G::FN + 16) * 8 + 2 * CT * (int)sizeof(CellInfo) + 2 * (int)sizeof(UnitInfo) +
         CT * D * 16 + 16;
}

template <int D, int N, int MODE>
__global__ void __launch_bounds__(256, HD_LINE_MINB) line_kernel(const __grid_constant__ CellParams p) {
  using G = CGeo<D, N>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const int CT = p.CT;
  const int CND = CT * G::ND;
  double *U = reinterpret_cast<double *>(smem_raw);
  double *ACC = U + CND;
  double *carry = ACC + CND;                                  // [CT][FN]
  double *stab = carry + CT * G::FN;                          // xi[8], w[8]
  CellInfo *info0 = reinterpret_cast<CellInfo *>(stab + 16);  // [2][CT]
  UnitInfo *uinfo = reinterpret_cast<UnitInfo *>(info0 + 2 * CT);
  int4 *fbuf = reinterpret_cast<int4 *>((reinterpret_cast<uintptr_t>(uinfo + 2) + 15) & ~uintptr_t(15));
  const int tid = threadIdx.x, nth = blockDim.x;
  if (tid < 8) {
    stab[tid] = tid < N ? c_tab[N].xi[tid] : 0.0;
    stab[8 + tid] = tid < N ? c_tab[N].w[tid] : 0.0;
  }
  if ((int)blockIdx.x >= p.nunits) return;

  const size_t cs = p.pencil ? (size_t)p.lstride[1] : 1;
  auto copy_cells = [&](int first_cell) {
    if constexpr (G::ND % 2 == 0) {
      for (int i = tid; i < (CND >> 1); i += nth) {
        const int e = 2 * i, kc = e / G::ND, x = e - kc * G::ND;
        cp_async16(U + e, p.u + ((size_t)first_cell + kc * cs) * G::ND + x);
      }
    } else {
      for (int i = tid; i < CND; i += nth) {
        const int kc = i / G::ND, x = i - kc * G::ND;
        cp_async8(U + i, p.u + ((size_t)first_cell + kc * cs) * G::ND + x);
      }
    }
  };
  auto first_cell = [&](int uu, int g, const UnitInfo &ui) {
    return p.pencil ? ui.base + step_group(p, g, ui.dir0, ui.skew) : uu * CT;
  };
  auto decode_group = [&](int uu, int g, const UnitInfo &ui, CellInfo *inf) {
    for (int idx = tid; idx < CT * D; idx += nth) {
      const int kk = idx / D, i = idx - kk * D;
      decode_cell<D>(p, ui, uu, g, kk, inf[kk], i);
      const int pf = inf[kk].pflag[i];
      if (pf >= 0) cp_async16(fbuf + idx, p.flags + (pf & ~3));
    }
    cp_async_commit();
  };
  auto resolve_group = [&](CellInfo *inf) {
    for (int idx = tid; idx < CT * D; idx += nth) {
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
    __syncthreads();  // previous group done: U, ACC, carry reads, info[s ^ 1] are free
    if (prev_unit >= 0 && tid == nth - 1) {
      __threadfence();
      *(volatile int *)(p.flags + prev_unit) = p.epoch | (prev_step + 1);
    }
    if (p.pencil && gi == 0 && ju > 0) {
      const int u2 = u + gridDim.x;
      if (tid < D && u2 < p.nunits) decode_unit<D>(p, u2, tid, uinfo[(ju + 1) & 1]);
    }
    copy_cells(first_cell(u, gi, uinfo[ju & 1]));
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();  // the cells (and the next unit's decode)
    const UnitInfo &ui_next = uinfo[(ju + (gn == 0 ? 1 : 0)) & 1];
    line_pass<D, N, MODE, 0>(p, info, stab, U, ACC, carry, tid, nth);
    if constexpr (D > 2) {
      __syncthreads();
      line_pass<D, N, MODE, 1>(p, info, stab, U, ACC, carry, tid, nth);
    }
    if constexpr (D > 3) {
      __syncthreads();
      line_pass<D, N, MODE, (D > 3 ? 2 : 0)>(p, info, stab, U, ACC, carry, tid, nth);
    }
    if constexpr (D > 4) {
      __syncthreads();
      line_pass<D, N, MODE, (D > 4 ? 3 : 0)>(p, info, stab, U, ACC, carry, tid, nth);
    }
    if constexpr (D > 5) {
      __syncthreads();
      line_pass<D, N, MODE, (D > 5 ? 4 : 0)>(p, info, stab, U, ACC, carry, tid, nth);
    }
    __syncthreads();
    if (has_next) decode_group(un, gn, ui_next, info0 + (s ^ 1) * CT);
    line_pass<D, N, MODE, D - 1>(p, info, stab, U, ACC, carry, tid, nth);
    cp_async_wait<0>();
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
    if (tid == nth - 1) {
      __threadfence();
      *(volatile int *)(p.flags + prev_unit) = p.epoch | (prev_step + 1);
    }
  }
}

}  // namespace hd
