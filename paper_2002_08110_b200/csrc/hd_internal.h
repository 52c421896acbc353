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

// x-space partition of the ranks (hd_plan.cpp)
struct Partition {
  int d = 0, d_x = 0, P = 1, rank = 0;
  int xparts[3] = {1, 1, 1};  // ranks per x dim
  int bcoord[3] = {0, 0, 0};  // this rank's block coordinates
  long long off[6] = {0, 0, 0, 0, 0, 0}, len[6] = {1, 1, 1, 1, 1, 1};  // local box of the global cell grid
  long long ncells_local = 0;
};
// halo of one x dim (hd_plan.cpp): what crosses the rank faces along it
struct HaloDim {
  bool active = false;
  int left = 0, right = 0;             // neighbour ranks along the dim
  std::vector<int> send_left;          // local cells (low face, a_i < 0) whose traces go to the left rank
  std::vector<int> send_right;         // local cells (high face, a_i > 0) whose traces go to the right rank
  long long n_from_left = 0, n_from_right = 0;  // traces received (positions with a_i > 0 / a_i < 0)
  std::vector<int> slot;               // per face-plane position: slot in the receive buffer
};
int host_cell_sign(const hd_mesh_desc &ds, const double *h, int d, int i, const long long *cg);
bool make_partition(const hd_mesh_desc &ds, Partition &pt, std::string &err);
void make_halo(const hd_mesh_desc &ds, const Partition &pt, const double *h, int i, HaloDim &hd);

// Kernel parameters of the fused cell kernel (passed by value as __grid_constant__).
// Work decomposition: pencil mode -- a group = CT cells at one dim-0 position from CT
// adjacent pencils (CT | L_1), a unit = those CT pencils, one group per step; multi-pencil mode (small
// d) -- a group = CT consecutive cells holding whole pencils, one group per unit.
struct CellParams {
  const double *u;        // operator input (never written by the kernel)
  double *out;            // A-mode: v; RK-mode: U_new
  double *du;             // RK-mode: dU (read unless first stage, written)
  int mode;
  int epoch;              // launch epoch << 10: a unit flag holds epoch | (groups completed in this launch)
  double rk_a, rk_b;      // stage coefficients A_s, B_s
  double dtfac;           // 1 (A-mode) or dt (RK-mode): folded into the line speeds
  double jdet;            // |J| = prod h_i
  int nunits;             // units of this launch
  int CT;                 // cells per group
  int GPU;                // groups (steps) per unit
  int UC;                 // cells per unit (trace-buffer slot size)
  int FN;                 // n^(d-1): doubles per trace
  int ND;                 // n^d: doubles per cell
  int prefetch;           // bulk-prefetch neighbour cells that will be read directly into L2
  int line;               // 1: line kernel (hd_line.cuh; face layout = line index), 0: tile kernel
  int pencil;             // 1: pencil mode
  int pubany;             // some dim publishes traces (unit flags needed)
  int L[kMaxD];           // cells per dim (local box)
  int lstride[kMaxD];     // cell-index stride per dim (memory order)
  int ustride[kMaxD];     // unit-index stride per dim (pencil mode, dims >= 1)
  double lo[kMaxD], h[kMaxD], inv_h[kMaxD];
  double a_const[kMaxD];
  double a_lin[kMaxD][kMaxD];
  int pub[kMaxD];         // 1: dim publishes traces into tbuf (one slot per unit) for its downwind neighbour
  int follow[kMaxD];      // pencil mode, dims >= 1: traversal follows the sign of a_i (depends on slower dims only)
  int skew;               // pencil mode: a pencil starts at group (-skew * sum_j t_j) mod GPU (pencil_decode)
  int discard;            // drop consumed published-trace lines from L2 (no write-back)
  int dbg;                // timing experiments only (HD_DBG; wrong results): 1 no direct reads, 2 no stores,
                          // 4 no trace publication
  int pubmode;            // how progress flags are released (publish_flag)
  double *tbuf[kMaxD];    // trace storage per dim: [unit][cell in unit][n^(d-1)]
  int *flags;             // [nunits] unit completion flags (value = epoch)
  // multi-rank: the local box starts at global cell coordinates coff; along a split x dim
  // a neighbour outside the box is on another rank and its trace comes from the halo buffer
  int coff[kMaxD];
  int xsplit[kMaxD];
  const double *hbuf[kMaxD];  // received traces per x dim: [slot][n^(d-1)]
  const int *hslot[kMaxD];    // face-plane position -> slot
};

// Halo pack (hd_kernels.cu): traces of the listed cells (entry e: cell index, dim, sign) into
// out[e][n^(d-1)], face points in the consumer's phase layout.
struct PackParams {
  int line;             // face layout of the consuming kernel (1: line index)
  const double *u;
  double *out;
  const int *cells;     // [nent]
  const int *dimsg;     // [nent]: dim | (sign << 8)
  long long nent;
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
  long long off[kMaxD], len[kMaxD];  // local box in the global cell grid
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
cudaError_t launch_pack_kernel(int d, int n, const PackParams &p, cudaStream_t s, long long *launches);
bool cell_kernel_supported(int d, int n);
// Kernel geometry for (d, n) on a local box with L0 cells along dim 0 and ncells cells: cells per group
// CT, pencil mode, threads per CTA, dynamic smem bytes, phases.
struct CellGeometry {
  int CT, pencil, GPU, threads, smem, phases, line;
};
CellGeometry cell_geometry(int d, int n, int L0, int L1, long long ncells, int line, int pencil_ok);
cudaError_t cell_grid_size(int d, int n, const CellGeometry &g, int sms, int *grid);

}  // namespace hd

namespace hd {
struct NcclApi;  // dlopen'ed NCCL entry points (hd_api.cpp)
}

struct hd_mesh {
  hd_mesh_desc desc;
  int d, n;
  long long nd;            // n^d
  long long ncells_global, ncells_local;
  long long cx_total, cx_begin, cx_end;  // flat x-cell range of the local box (-1: not contiguous)
  long long owned_dofs;
  hd::Partition pt;        // local box and rank grid
  double h[6];
  double jdet;
  hd::Tables1D tab;
  int device, sms;
  long long launches;
  // trace machinery (device buffers owned by the mesh)
  hd::CellGeometry geo;
  int nunits;
  int pub[6], follow[6];
  double *tbuf[6];
  int *flags;
  long long epoch;
  int grid;
  // halo (nranks > 1): per x dim receive buffer and slot table; one send buffer for all dims, laid
  // out per dim as [to the right rank][to the left rank]
  hd::HaloDim halo[3];
  double *hbuf[3];
  int *hslot[3];
  long long send_off_right[3], send_off_left[3];  // entry offsets into the send buffer
  long long nsend;                                // entries
  int *pack_cells, *pack_dimsg;
  double *sendbuf;
  void *nccl_comm;         // ncclComm_t when the NCCL transport is used
};
