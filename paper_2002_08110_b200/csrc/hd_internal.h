// hd_internal.h -- host/device shared definitions of the product library (not the C ABI).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/hd.h"

namespace hd {

constexpr int kMaxD = 6;
constexpr int kMaxN = 6;

// 1D tables for n nodes: everything the cell kernel needs from the
// reference interval. Computed on the host in long double (hd_tables.cpp).
struct Tables1D {
  double xi[kMaxN];          // Gauss-Legendre nodes on [0,1]
  double w[kMaxN];           // weights (sum 1)
  // merged 1D operator for unit speed, upwind, by sign s (0: a > 0, 1: a < 0):
  //   (L u)_m = sum_q K[s][m][q] u_q + lam[s][m] * (sum_q tau[s][q] u^nb_q)
  // s = 0: nb = left neighbour,  K = (w_q l'_m(xi_q) - l_m(1) l_q(1)) / w_m, lam = l_m(0)/w_m,  tau = l_q(1)
  // s = 1: nb = right neighbour, K = (w_q l'_m(xi_q) + l_m(0) l_q(0)) / w_m, lam = -l_m(1)/w_m, tau = l_q(0)
  double K[2][kMaxN][kMaxN];
  double lam[2][kMaxN];
  double tau[2][kMaxN];
};

// Host-side computation of the tables (independent of the oracle).
void build_tables(int n, Tables1D &t);

enum Mode : int { kModeAdvection = 0, kModeRK = 1, kModeRKFirst = 2 };

// Trace mode of a dimension:
//   kTraceNone: every consumer reads its upwind neighbour cell and forms the trace itself
//   kTraceRing: producers publish downwind traces into an L2-resident ring of items
//   kTraceFar : producers publish into a full-size buffer (consumer is many items later)
enum TraceMode : int { kTraceNone = 0, kTraceRing = 1, kTraceFar = 2 };

// Kernel parameters (passed by value as __grid_constant__).
struct CellParams {
  const double *u;        // operator input (never written by the kernel)
  double *out;            // A-mode: v; RK-mode: U_new
  double *du;             // RK-mode: dU (read unless first stage, written)
  int ncells;             // owned cells (< 2^31)
  int nitems;             // work items = ncells / C (C consecutive cells along dim 0)
  int mode;
  int target;             // flag value that marks "published in this launch" (epoch * warps per item)
  double rk_a, rk_b;      // stage coefficients A_s, B_s
  double dtfac;           // 1 (A-mode) or dt (RK-mode): folded into the line speeds
  double jdet;            // |J| = prod h_i
  // geometry (local box of cells)
  int L[kMaxD];           // cells per dim
  int IL[kMaxD];          // item-grid extents (IL[0] = L[0] / C)
  int istride[kMaxD];     // item-index stride per dim (traversal order)
  int lstride[kMaxD];     // cell-index stride per dim (memory order)
  double lo[kMaxD], h[kMaxD], inv_h[kMaxD];
  double a_const[kMaxD];
  double a_lin[kMaxD][kMaxD];
  // upwind traces
  int tmode[kMaxD];       // TraceMode per dim
  int dirneg[kMaxD];      // traversal direction of trace dims: 1 if a_i < 0 everywhere
  int rmask[kMaxD];       // ring slots - 1 (kTraceRing)
  double *tbuf[kMaxD];    // trace storage per dim: [slot][cell in item][n^(d-1)]
  int *flags;             // [nitems][phases + 1] publication counters
  int pubmask;            // bit ph: phase ph's counter is waited on (publish it)
  int debug;
};

// Stream kernels
struct StreamParams {
  double *u;
  long long ndofs;
  double jdet;
  int inverse;
};

struct FillParams {
  double *u;
  long long ncells;
  long long nx_local, cx_begin;
  long long L[kMaxD];
  double lo[kMaxD], h[kMaxD];
  int d_x, d;
  int recipe;
  unsigned long long seed;
};

// Launchers (hd_kernels.cu). Return cudaError_t of the launch; *launches incremented.
cudaError_t upload_tables(int n, const Tables1D &t);
cudaError_t launch_cell_kernel(int d, int n, const CellParams &p, cudaStream_t s, long long *launches, int grid);
cudaError_t launch_mass_kernel(int d, int n, const StreamParams &p, cudaStream_t s, long long *launches, int sms);
cudaError_t launch_fill_kernel(int d, int n, const FillParams &p, cudaStream_t s, long long *launches);
bool cell_kernel_supported(int d, int n);
// Kernel geometry for (d, n, L0): cells per item C (a divisor of L0), threads per CTA, phases,
// warps per item, and the persistent grid size (co-resident CTAs).
struct CellGeometry {
  int C, threads, phases, warps_per_item, smem;
};
CellGeometry cell_geometry(int d, int n, int L0);
cudaError_t cell_grid_size(int d, int n, int L0, int mode, int sms, int *grid);

}  // namespace hd

struct hd_mesh {
  hd_mesh_desc desc;
  int d, n;
  long long nd;            // n^d
  long long ncells_global, ncells_local;
  long long cx_total, cx_begin, cx_end, nx_local, nv;
  long long owned_dofs;
  double h[6];
  double jdet;
  hd::Tables1D tab;
  int device, sms;
  long long launches;
  // trace machinery (device buffers owned by the mesh)
  hd::CellGeometry geo;
  int tmode[6], rmask[6], dirneg[6];
  double *tbuf[6];
  int *flags;
  long long epoch;
  int grid;
};
