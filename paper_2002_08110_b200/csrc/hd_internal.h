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
constexpr int kMaxChunk = 8;  // v-chunks of a pipelined multi-rank stage

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
  double Dw[kMaxN][kMaxN];   // w_q l'_m(xi_q): the unscaled weak volume derivative (FCL path)
};

// Host-side computation of the tables (independent of the oracle).
void build_tables(int n, Tables1D &t);
// GLL <-> Gauss basis-change matrices (hd_tables.cpp): [kind][out * n + in], kind as hd_basis_kind
void build_basis_tables(int n, double S[4][kMaxN * kMaxN]);

// basis_kernel (hd_basis.cu): the 1D matrix S applied along every dim of every cell
struct BasisParams {
  const double *u;
  double *v;
  long long ncells;
  int d, cb, nbuf;           // dims, cells per CTA batch, staging buffers (2: next batch prefetched)
  double S[kMaxN * kMaxN];   // [out * n + in]
};

enum Mode : int { kModeAdvection = 0, kModeRK = 1, kModeRKFirst = 2, kModeAdvAcc = 3 /* v += A u (central flux) */ };

// x-space partition of the ranks (hd_plan.cpp)
struct Partition {
  int d = 0, d_x = 0, P = 1, rank = 0;
  int parts[6] = {1, 1, 1, 1, 1, 1};   // ranks per dim (x dims, then v dims)
  int bcoord[6] = {0, 0, 0, 0, 0, 0};  // this rank's block coordinates
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

// Static schedule of the fused cell kernel (built on the host by hd_sched.cpp, read by the kernel): one
// record per (group, cell slot k, dim i), 32 bytes. A group is the CT cells one CTA processes together;
// groups are numbered unit * GPU + step. Everything about a cell and its upwind traces is decided here
// once per mesh -- the kernel does no index decoding. The one run-time decision left is whether a
// published trace is ready (the producer's progress flag), which falls back to a direct read.
enum TraceSrc : unsigned char { kSrcDirect = 0, kSrcGroup = 1, kSrcCarry = 2, kSrcPub = 3, kSrcHalo = 4 };
enum TraceOut : unsigned char { kOutNone = 0, kOutCarry = 1, kOutPub = 2 };
struct SchedDim {
  double base;            // a_i at the cell's lower corner (global coordinates; speed of the cell's lines
                          // before the per-node offsets); the sign below is that of a_i on the cell
  int nb;                 // upwind neighbour cell (local index): kSrcDirect, and the fallback of kSrcPub
  int slot;               // kSrcGroup: neighbour slot k' in the group; kSrcPub: producer trace slot;
                          // kSrcHalo: receive-buffer slot
  int pflag;              // kSrcPub: producer unit whose progress flag is checked (-1: none)
  int need;               // kSrcPub: producer steps (flag payload) that must be complete
  unsigned char src, out, sg, pad;  // TraceSrc, TraceOut, 1: a_i < 0 (upwind neighbour at +e_i)
  int pad2;
};
// per (group, cell slot): the cell and the slot its published traces go to
struct SchedCell {
  int cell;               // local cell index (memory order)
  int oslot;              // kOutPub: trace slot of this cell (same index in every dim's buffer)
};
static_assert(sizeof(SchedDim) == 32, "SchedDim is 32 bytes");

// Kernel parameters of the fused cell kernel (passed by value as __grid_constant__; > 4 KB, which
// CUDA >= 12.1 allows). Work decomposition: a group = CT cells (pencil mode: one dim-0
// position of CT adjacent pencils; else CT consecutive cells), a unit = GPU groups processed in order by
// one CTA; units are dealt round-robin to the persistent CTAs.
struct CellParams {
  const double *u;        // operator input (never written by the kernel)
  double *out;            // A-mode: v; RK-mode: U_new
  double *du;             // RK-mode: dU (read unless first stage, written)
  int mode;
  int epoch;              // launch epoch << 10: a unit flag holds epoch | (groups completed in this launch)
  double rk_a, rk_b;      // stage coefficients A_s, B_s
  double dtfac;           // 1 (A-mode) or dt (RK-mode): folded into the line speeds
  double jdet;            // |J| = prod h_i
  int nunits;             // units of the mesh
  int u_begin, u_end;     // units of this launch (all, or one v-chunk of a pipelined multi-rank stage)
  int CT;                 // cells per group
  int GPU;                // groups (steps) per unit
  int ND;                 // n^d: doubles per cell
  int FN;                 // n^(d-1): doubles per trace
  int prefetch;           // bulk-prefetch cells that will be read directly into L2
  long long cstride;      // cell-index stride between the cells of a group (pencil mode: L_0; else 1)
  const SchedDim *sched;  // [nunits * GPU][CT][D]
  const SchedCell *schedc;  // [nunits * GPU][CT]
  int *flags;             // [nunits rounded up to 4] unit progress flags
  int *uctr;              // unit counter of the launch (dynamic unit dealing; zeroed before every launch)
  int slab;               // > 1: slab super-units -- dim-1 published traces are this CTA's own (L2 evict_last,
                          // discarded once read)
  double *tbuf[kMaxD];    // published traces per dim: [slot][n^(d-1)]
  const double *hbuf[kMaxD];  // received halo traces per x dim: [slot][n^(d-1)]
  int var[kMaxD];         // 1: a_i depends on z (line speeds vary: u is scaled per line); 0: constant
  double inv_h[kMaxD], h[kMaxD], lo[kMaxD];
  double a_const[kMaxD];
  double a_lin[kMaxD][kMaxD];
  double fac[kMaxD];      // dtfac / h_i (line speed = (a_i at the line) * fac)
  double slin[kMaxD][kMaxD];  // a_lin[i][j] h_j fac_i: change of the line speed of dim i per unit node of dim j
  int coff[kMaxD];        // global cell coordinates of the local box origin (pack kernel)
  int L[kMaxD];           // local box (pack kernel)
  // HD_DEBUG builds only: error word (bit 1 index out of range, bit 2 stale halo trace,
  // bit 4 non-finite value), bounds, and the halo freshness tags: stag[dim][dir] = epoch of the
  // traces this rank packed, rtag[dim][dir] = epoch of the traces it received (dir 0: from / to the left
  // neighbour's a_i > 0 side, 1: a_i < 0)
  int *err;
  int *stag;
  const int *rtag;
  long long ncells;
  long long nhalo[kMaxD];
  // constant-speed dims: s_i K[s] and s_i tau[s] with s_i = a_i dtfac / h_i (compact [dim][sign][N][N]
  // and [dim][sign][N] for the mesh's N); variable dims use the unit-speed c_tab tables on scaled lines
  double Ks[kMaxD * 2 * kMaxN * kMaxN];
  double Ts[kMaxD * 2 * kMaxN];
};

// Halo pack (hd_kernels.cu): traces of the listed cells (entry e: cell index, dim, sign) into
// out[e][n^(d-1)], face points in the consumer's phase layout.
struct PackParams {
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

// Face-centric loop (FCL) comparison path of v <- A(u) (hd_fcl.cu).
struct FclParams {
  const double *u;
  double *v;
  double *tr;             // [d][2][ncells][n^(d-1)]: face traces u(xi_i = side)
  double *G;              // [d][ncells][n^(d-1)]: flux of the face (cell, cell + e_i) times |J|/h_i w_f
  long long ncells;
  long long L[kMaxD];     // cells per dim (single rank: the global grid)
  unsigned L32[kMaxD];    // the same as 32-bit divisors (cell indices fit 31 bits)
  double lo[kMaxD], h[kMaxD], jdet_h[kMaxD];  // jdet_h[i] = |J| / h_i
  double a_const[kMaxD];
  double a_lin[kMaxD][kMaxD];
  double xi[kMaxN], w[kMaxN], l0[kMaxN], l1[kMaxN];
  double Dw[kMaxN][kMaxN];  // w_q l'_m(xi_q)
  int flux;               // 0 upwind, 1 central
  // Vlasov-Poisson (NEXT-1): when E is set, a_{d_x + l} -= E[l][x cell][x node] (P:3963 a = (v, -E(x)))
  const double *E;
  int d_x;
  long long ncx;          // x cells (the flat x-cell index is cell % ncx: x dims are the fastest)
  int nx;                 // n^d_x x nodes per x cell
};
// Vlasov-Poisson field pipeline (hd_fcl.cu): rho = 1 - int f dv, its Fourier coefficients, E = -grad phi
struct VpParams {
  int d_x, n, nx, nv, ND;     // nx = n^d_x, nv = n^d_v, ND = n^d
  long long ncx, ncv;         // x cells, v cells
  long long Lx[3];            // x cells per x dim
  double lo[3], h[3], Lbox[3], xi[kMaxN], w[kMaxN];
  double vol_x;               // |Omega_x|
  long long K[3], nmodes;     // modes |m_i| <= K_i, prod (2 K_i + 1)
  double wv[216];             // per v node: prod w_{j_v} h_v (|J_v| times the v quadrature weight)
};
cudaError_t launch_vp_fields(const VpParams &p, const double *f, double *rho, double *rhohat, double *E, cudaStream_t s,
                             long long *launches, int sms);
cudaError_t launch_vp_update(double *U, double *dU, const double *w, long long n, double A, double B, double dt,
                             int first, cudaStream_t s, long long *launches, int sms);
bool fcl_supported(int d, int n);
// three launches (cell, face, lift); *launches += 3
cudaError_t launch_fcl(int d, int n, const FclParams &p, cudaStream_t s, long long *launches, int sms);

// Launchers (hd_kernels.cu). Return cudaError_t of the launch; *launches incremented.
cudaError_t upload_tables(int n, const Tables1D &t);
cudaError_t launch_cell_kernel(int d, int n, const CellParams &p, cudaStream_t s, long long *launches, int grid);
cudaError_t launch_mass_kernel(int d, int n, const StreamParams &p, cudaStream_t s, long long *launches, int sms);
cudaError_t launch_fill_kernel(int d, int n, const FillParams &p, cudaStream_t s, long long *launches);
cudaError_t launch_pack_kernel(int d, int n, const PackParams &pp, const CellParams &cp, cudaStream_t s,
                               long long *launches);
// HD_DEBUG: set bit 4 of *err if any of the n values is not finite
cudaError_t launch_finite_check(const double *v, long long n, int *err, cudaStream_t s);
bool cell_kernel_supported(int d, int n);
cudaError_t launch_basis_kernel(int n, BasisParams &p, cudaStream_t s, long long *launches, int sms);
bool basis_kernel_supported(int d, int n);

// Static schedule of a mesh (hd_sched.cpp): [nunits * GPU][CT][d] records (see SchedDim).
// forced = -1: upwind by the sign of a_i; 0 / 1: every dim takes its left / right neighbour (central flux)
void build_schedule(const hd_mesh &m, std::vector<SchedDim> &out, std::vector<SchedCell> &cells, int forced);
// Kernel geometry for (d, n) on a local box with L0 cells along dim 0 and ncells cells: cells per group
// CT, pencil mode, threads per CTA, dynamic smem bytes, phases.
struct CellGeometry {
  int CT, pencil, GPU, threads, smem, phases;
};
CellGeometry cell_geometry(int d, int n, int L0, int L1, long long ncells, int pencil_ok);
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
  // slab super-units: the kernel runs `slab` consecutive pencil units (the pencils of one
  // dim-0/dim-1 slab, dim-1 traversal order) as one unit of slab * GPU steps; 1 = pencil units
  int slab;
  int pub[6], follow[6];
  int skew;                // pencil mode: a unit starts at step (-skew * sum_j t_j) mod GPU (hd_sched.cpp)
  double *tbuf[6];
  int *flags;
  long long nflags;        // flag words allocated (nunits rounded up to 4)
  hd::SchedDim *sched;     // device copy of the static schedule (central flux: the left-neighbour one)
  hd::SchedCell *schedc;
  hd::SchedDim *sched2;    // central flux: the right-neighbour schedule
  hd::SchedCell *schedc2;
  long long epoch;
  int grid;
  // halo (nranks > 1): per x dim receive buffer and slot table; one send buffer for all dims, laid
  // out per dim as [to the right rank][to the left rank]
  hd::HaloDim halo[6];
  double *hbuf[6];
  int *hslot[6];
  long long nsend;                                // entries of the send list (chunk-major)
  // v-chunk pipeline of a multi-rank stage: chunk c = the units [chunk_u[c], chunk_u[c+1]),
  // i.e. the cells whose slowest (v) coordinate lies in one range. Per chunk: its send-list entries
  // [pe0, pe1) and, per x dim, (offset, count) of the traces sent to the right / left rank (entries of the
  // send list) and received from the left / right rank (slots of hbuf[i]).
  int nchunk;
  int chunk_u[hd::kMaxChunk + 1];
  struct ChunkHalo {
    long long pe0, pe1;
    long long sr[6][2], sl[6][2], rl[6][2], rr[6][2];
    long long srq[6], slq[6];  // first entry of the chunk's part of the dim's send_right / send_left list
  } chunk[hd::kMaxChunk];
  cudaStream_t comm;                              // NCCL transport: pack + exchange stream
  int *dbg;                                       // HD_DEBUG: [0] error word, [1..12] stag, [13..24] rtag
  cudaEvent_t ev_u, ev_chunk[hd::kMaxChunk];
  int *pack_cells, *pack_dimsg;
  double *sendbuf;
  void *nccl_comm;         // ncclComm_t when the NCCL transport is used
  double *fcl_tr, *fcl_G;  // FCL comparison path buffers (allocated by the first hd_apply_advection_fcl)
  double *vp_rho, *vp_rhohat, *vp_E;  // Vlasov-Poisson field buffers (allocated by the first hd_vp_* call)
};
