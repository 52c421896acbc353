/* hd.h -- C ABI of the B200-native DG advection hot path of hyper.deal (arXiv 2002.08110).
 *
 * Citations: P:n = PAPER.md line n, S:n = SPEC.md line n (the paper text and the spec written
 * from it); Cn = reading n of DESIGN.md "Readings".
 *
 * What the library computes (FP64, periodic Cartesian box T = T_x (x) T_v; nodal
 * Lagrange basis on the n = k+1 Gauss-Legendre points of each 1D reference interval [0,1],
 * reading C1; upwind numerical flux, or the central flux on single-rank meshes, reading C3):
 *   hd_apply_advection  v <- A(u), the DG weak form of Eq. into:adv:ref,
 *                       A(u)_i = (grad phi_i, a u)_cell - sum_faces <phi_i, (a.n) u_up>_face
 *                       (sign convention P:236, reading C4; output is the weak form, C5).
 *   hd_apply_inv_mass   u <- M^-1 u in place (P:3, "u <- M(u)" read as M^-1, C6;
 *                       Alg. 2 step 4 P:1095-1097, with |J| restored, C7). Collocated mass is
 *                       diagonal: M_qq = |J| prod_i w_{q_i} (C2).
 *   hd_apply_mass       u <- M u in place (test aid).
 *   hd_rk_step          nsteps steps of the five-stage fourth-order low-storage Runge-Kutta
 *                       method in the Williamson 2N form (reading C13)
 *                       with the merged operator M^-1 A as right-hand side.
 *   hd_fill_initial     the seeded synthetic initial data of DESIGN.md "Inputs" (reading C14).
 *
 * Data layout (reading C19): a DoF vector holds this rank's owned cells; cell-local DoF
 * j = sum_i m_i n^i (dim 0 = x_1 fastest ... last v dim slowest); owned cells in the order
 * [c_v][c_x - cx_begin], c_x and c_v lexicographic with the first axis fastest. With nranks = 1
 * this is the global order g = c_v |C_x| + c_x. Each cell occupies n^d consecutive
 * doubles; vectors must be 16-byte aligned device memory (HD_ERR_ARG otherwise; cudaMalloc and torch
 * allocations are 256-byte aligned).
 *
 * Ownership: every DoF vector is caller-allocated device memory of hd_mesh_info's owned_dofs
 * doubles. The mesh owns its constant tables, halo plan and buffers, NCCL communicator and
 * internal events; hd_destroy_mesh frees them.
 *
 * Streams: all work is enqueued on the given CUDA stream (cudaStream_t passed as void*; NULL =
 * legacy default stream); calls return without host synchronisation unless stated.
 *
 * Errors: every call returns an hd_status; no exception crosses the ABI. hd_last_error() gives a
 * thread-local message for the last non-OK status of the calling thread. Asynchronous CUDA
 * faults surface on a later call as HD_ERR_CUDA. A mesh is not re-entrant (one thread at a time).
 */
#ifndef HD_H
#define HD_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hd_mesh hd_mesh;

typedef enum {
  HD_OK = 0,
  HD_ERR_ARG = -1,         /* invalid argument (dims, k, cells, box, field, aliasing, null) */
  HD_ERR_UNSUPPORTED = -2, /* valid but not built for the GPU path (see hd_create_mesh) */
  HD_ERR_CUDA = -3,        /* CUDA runtime error (message in hd_last_error) */
  HD_ERR_NCCL = -4,        /* NCCL error (multi-rank halo) */
  HD_ERR_OOM = -5,         /* device or host allocation failed */
  HD_ERR_STATE = -6        /* call not allowed in the current state */
} hd_status;

typedef struct {
  int d_x, d_v;         /* space dims, 1..3 each; d = d_x + d_v in 2..6 */
  int k;                /* polynomial degree; n = k+1 in 2..6; n^d must be <= 4096 on the GPU path */
  long long cells[6];   /* cells per dim, x dims first; all >= 1 */
  double lo[6], hi[6];  /* box per dim, hi > lo; periodic in every dim (C9) */
  double a_const[6];    /* advection field a_i(z) = a_const[i] + sum_j a_lin[i][j] z_j ...   */
  double a_lin[36];     /* ... row-major [i][j]; a_lin[i][i] must be 0 (divergence free); the
                           sign of a_i must be constant on every cell with the upwind flux
                           (reading C11; HD_ERR_UNSUPPORTED otherwise) */
  int flux;             /* 0 = upwind; 1 = central, F* = (a.n)(u- + u+)/2, nranks = 1 only
                           (HD_ERR_UNSUPPORTED otherwise); evaluated as the mean of the two one-sided
                           operators (every face taking its left cell's trace, resp. its right cell's),
                           i.e. two cell-kernel launches per application or RK stage */
  int rank, nranks;     /* phase-space partition over nranks ranks: the ranks form a grid
                           parts[0] x .. x parts[d-1] over the cells (parts = xparts, then vparts); rank r
                           has block coordinates b_i = (r / prod_{j<i} parts_j) % parts_i */
  const void *nccl_id;  /* 128-byte ncclUniqueId when nranks > 1 and the NCCL transport is wanted; NULL
                           selects the in-process loopback transport (hd_*_group calls) */
  int xparts[3];        /* ranks per x dim (p_i must divide cells[i]); all of xparts and vparts 0 =
                           automatic: the x factorisation with the smallest halo, x-slabs on ties */
  int vparts[3];        /* ranks per v dim (checkerboard x-v partition; 0 or 1 = not split).
                           Explicit partitions need prod(xparts) * prod(vparts) = nranks */
} hd_mesh_desc;

/* Validate desc, build the 1D tables and the partition. HD_ERR_ARG for invalid input (S:48:
 * invalid dim or zero subdivision; DoF-count overflow S:74); HD_ERR_UNSUPPORTED for a valid mesh
 * outside the built kernel set. *out receives an opaque mesh; desc is copied. */
hd_status hd_create_mesh(const hd_mesh_desc *desc, hd_mesh **out);
hd_status hd_destroy_mesh(hd_mesh *m);

/* owned_dofs: length of this rank's DoF vectors; [cx_begin, cx_end): owned range of the
 * flattened x-cell index c_x. Any output pointer may be NULL. */
hd_status hd_mesh_info(const hd_mesh *m, long long *owned_dofs, long long *cx_begin, long long *cx_end);

/* The rank's local box of the global cell grid: off[i], len[i] per dim (d entries used) and the x part of the
 * rank grid xparts[3] (the v part is cells[i] / len[i]). Local vectors hold the box's cells
 * lexicographically (first axis fastest). Any output pointer may be NULL. */
hd_status hd_mesh_box(const hd_mesh *m, long long *off, long long *len, int *xparts);

/* v <- A(u) (weak form). u, v: device vectors of owned_dofs doubles that must not overlap
 * (HD_ERR_ARG otherwise). t is the evaluation time (the built fields do not depend on t). */
hd_status hd_apply_advection(hd_mesh *m, const double *u, double *v, double t, void *stream);

/* v <- A(u) through the face-centric loop (FCL) the paper compares against its element-centric default
 * (SURVEY §8(f) NEXT-3): a cell pass (volume term and both face traces of every dim),
 * a face pass (each face's numerical flux computed once, upwind or central by desc.flux) and a
 * lift pass (the flux tested on both sides). Same result as hd_apply_advection up to rounding order.
 * u, v: non-overlapping device vectors of owned_dofs doubles (HD_ERR_ARG otherwise). The first call
 * allocates the mesh's face buffers, 3 d n^(d-1) doubles per cell (HD_ERR_OOM if they do not fit; freed by
 * hd_destroy_mesh). Single-rank meshes whose cell fits 200 KB of shared memory (HD_ERR_UNSUPPORTED
 * otherwise). Three kernel launches on stream. */
hd_status hd_apply_advection_fcl(hd_mesh *m, const double *u, double *v, double t, void *stream);

/* Vlasov-Poisson (Eq. equ:vp:close; DESIGN.md §6 "Vlasov-Poisson"). A mesh
 * with d_x = d_v <= 3, one rank, whose field holds the x part a_i = v_i (a_lin[i][d_x + i] = 1); the v part of
 * the phase-space field is a_{d_x+l} = (desc field) - E_l(x), composed on the fly from an E table at the x
 * Gauss nodes. Errors as hd_apply_advection_fcl; HD_ERR_UNSUPPORTED for other meshes.
 *
 * hd_vp_fields: rho(x) = 1 - int f dv at every x node and E = -grad phi with -lap phi = rho on the
 *   periodic x box, solved spectrally (SPEC S:567-575 substitute for the paper's multigrid, reading C24):
 *   rhohat(m) = |Omega_x|^-1 (Gauss rule of rho_h e^{-i k.x}), |m_i| <= (cells_i - 1)/2, zero mode dropped.
 *   f: device vector of owned_dofs doubles. rho (ncx * n^d_x doubles, [x cell][x node], may be NULL) and
 *   E (d_x * ncx * n^d_x doubles, [component][x cell][x node], may be NULL): device outputs.
 * hd_apply_advection_vp: v <- A(u) (weak form) with a = (v, -E(x)) through the face-centric loop (the
 *   sign of -E changes inside cells, which the upwind ECL kernel does not allow, reading C11). E as above.
 * hd_vp_rk_step: nsteps LSRK(5,4) steps of df/dt = M^-1 A(f; E(f)) with E recomputed from every stage's f
 *   (S:577). buf[0] = f (updated in place), buf[1], buf[2] scratch: three distinct device vectors. */
hd_status hd_vp_fields(hd_mesh *m, const double *f, double *rho, double *E, void *stream);
hd_status hd_apply_advection_vp(hd_mesh *m, const double *u, const double *E, double *v, void *stream);
hd_status hd_vp_rk_step(hd_mesh *m, double *buf[3], double t, double dt, int nsteps, void *stream);

/* GLL nodal basis with Gauss quadrature: the paper's default discretisation and its
 * basis change ("a sequence of d 1D interpolation sweeps", Cartesian
 * part; DESIGN.md §6 "Basis change"). T[q][j] = l^GLL_j(xi^Gauss_q), applied along every dim of every cell.
 * The mesh's own vectors hold Gauss-point values (reading C1); these calls convert at the boundary.
 *
 * hd_basis_change: v <- (S x ... x S) u per cell, S by kind. u, v: device vectors of owned_dofs doubles, equal
 *   (in place) or non-overlapping (HD_ERR_ARG otherwise). Cell-local: any partition. One launch.
 * hd_apply_advection_gll: v <- A_L u = T^T A_G (T u), the weak form in the GLL basis (P:556-567 steps 1-5).
 *   work: device scratch of owned_dofs doubles; u, v, work pairwise non-overlapping. Errors as hd_apply_advection.
 * hd_rk_step_gll: hd_rk_step on GLL coefficients: buf[*sol] is converted to Gauss values in place, stepped,
 *   and the result converted back (T is constant in time, so no stage needs a basis change).
 * hd_basis_tables (host): gll[n] = the GLL points on [0,1]; T[4][n][n] = the matrices by kind, [out][in]. */
typedef enum {
  HD_GLL_TO_GAUSS = 0,   /* T       : GLL coefficients -> values at the Gauss points */
  HD_GAUSS_TO_GLL = 1,   /* T^-1    : Gauss values -> GLL coefficients */
  HD_GLL_TO_GAUSS_T = 2, /* T^T     : Gauss-basis weak form (test side) -> GLL-basis weak form */
  HD_GAUSS_TO_GLL_T = 3  /* T^-T */
} hd_basis_kind;
hd_status hd_basis_change(hd_mesh *m, const double *u, double *v, int kind, void *stream);
hd_status hd_apply_advection_gll(hd_mesh *m, const double *u, double *v, double *work, double t, void *stream);
hd_status hd_rk_step_gll(hd_mesh *m, double *buf[3], int *sol, double t, double dt, int nsteps, void *stream);
hd_status hd_basis_tables(int n, double *gll, double *T);

/* u <- M^-1 u and u <- M u, in place; one streaming pass, no communication. */
hd_status hd_apply_inv_mass(hd_mesh *m, double *u, void *stream);
hd_status hd_apply_mass(hd_mesh *m, double *u, void *stream);

/* nsteps (>= 1) LSRK(5,4) steps of size dt starting at time t. buf[0..2]: three distinct device
 * vectors; on entry buf[*sol] holds u^n, on exit buf[*sol] holds u^{n+nsteps} (the fused stage
 * cannot overwrite its operator input, so the solution rotates through the buffers). The other
 * two buffers are scratch and are overwritten. */
hd_status hd_rk_step(hd_mesh *m, double *buf[3], int *sol, double t, double dt, int nsteps, void *stream);

/* One fused stage s = 0..4 of the LSRK(5,4) step (the building block of hd_rk_step, exported for
 * stage-by-stage checks): dU <- A_s dU + dt M^-1 A(U) (s = 0: dU <- dt M^-1 A(U), dU not read), then
 * out <- U + B_s dU. U, dU, out: three distinct device vectors of owned_dofs doubles (HD_ERR_ARG if they
 * overlap); U is not written. Multi-rank meshes exchange the halo of U first (NCCL transport). */
hd_status hd_rk_stage(hd_mesh *m, const double *U, double *dU, double *out, int stage, double dt, void *stream);

/* Multi-rank meshes WITHOUT an NCCL communicator (desc.nccl_id == NULL): all P ranks' meshes live in
 * this process on the current device and the halo is moved by device copies (loopback transport, the
 * same buffer layout NCCL delivers). ms[r] must be rank r of P. u, v: P device vectors;
 * bufs: 3P device vectors (rank r uses bufs[3r .. 3r+2]); *sol as in hd_rk_step (common to all ranks). */
hd_status hd_apply_advection_group(hd_mesh **ms, int P, const double **u, double **v, double t, void *stream);
hd_status hd_rk_step_group(hd_mesh **ms, int P, double **bufs, int *sol, double t, double dt, int nsteps,
                           void *stream);

/* End-to-end variant with HOST buffers: copies u_host (owned_dofs doubles, ideally pinned) into
 * dbuf[0], runs nsteps steps, copies the solution back into u_out_host (may equal u_host), and
 * synchronises the stream before returning. dbuf: three distinct device scratch vectors. */
hd_status hd_rk_step_host(hd_mesh *m, const double *u_host, double *u_out_host, double *dbuf[3], double t,
                          double dt, int nsteps, void *stream);

/* u <- synthetic initial data: recipe 0 gauss2d, 1 uniform, 2 sines, 3 maxwellian (DESIGN.md
 * "Inputs"), counter-based in (seed, global DoF index), identical to the Python generator
 * paper_2002_08110_b200/inputs.py up to libm rounding. */
hd_status hd_fill_initial(hd_mesh *m, double *u, int recipe, unsigned long long seed, void *stream);

/* Host-only queries (no GPU needed), for inspection and tests of the host plan:
 * hd_tables_1d: the 1D tables the kernels use for n nodes (2..6): Gauss-Legendre nodes xi[n] and
 * weights w[n] on [0,1]; the merged unit-speed upwind line operator K[2][n][n], lift lam[2][n] and
 * neighbour-trace weights tau[2][n] (index 0: a > 0, left neighbour; 1: a < 0, right neighbour).
 * hd_lsrk_coefficients: the 2N coefficients A_s, B_s (s = 1..5) of hd_rk_step. */
hd_status hd_tables_1d(int n, double *xi, double *w, double *K, double *lam, double *tau);
hd_status hd_lsrk_coefficients(double *a, double *b);

/* Upwind-trace plan of the mesh per dimension (DESIGN.md §6 "Upwind trace sources"): tmode[i] = 0 (the
 * cell reads its upwind neighbour itself or gets it from the same CTA) or 2 (published into a full-size
 * buffer, one n^(d-1)-value slot per cell). Mode 1 (an L2-sized ring of slots) is reserved and not built:
 * ring_slots[i] is always 0. */
hd_status hd_mesh_traces(const hd_mesh *m, int *tmode, int *ring_slots);

/* 128-byte ncclUniqueId for hd_mesh_desc.nccl_id (rank 0 creates it and broadcasts it). Loads
 * libnccl.so.2 at run time; HD_ERR_NCCL if it is unavailable. */
hd_status hd_nccl_unique_id(void *out128);

/* Host-only plan queries (no GPU): the partition of desc->rank (xparts[3], off[6], len[6]) and its halo
 * lists along x dim `dim`: which = 0 traces sent to the left rank, 1 sent to the right rank (ids = global
 * ids of the RECEIVING cells, in message order), 2 received from the left rank, 3 from the right rank
 * (ids = global ids of this rank's receiving cells, in buffer order). *count: capacity of ids in, length
 * out (ids may be NULL to query the length); *peer: the partner rank (-1 if the dim is not split). */
hd_status hd_partition_info(const hd_mesh_desc *desc, int *xparts, long long *off, long long *len);
hd_status hd_halo_list(const hd_mesh_desc *desc, int dim, int which, long long *ids, long long *count, int *peer);

/* Host-only query of the v-chunk pipeline of desc->rank: *nchunk chunks; chunk_units[0..nchunk]
 * (may be NULL): chunk c = units [chunk_units[c], chunk_units[c+1]); plan (may be NULL; kMaxChunk = 8 x 6 x 8
 * long longs): for chunk c and split dim i, plan[(c*6+i)*8 + ...] = {first entry and count of the traces sent
 * to the right rank, as a range of hd_halo_list(which = 1); first entry and count of those sent to the left
 * rank (which = 0); first receive slot and count from the left rank; first receive slot and count from the
 * right rank}. */
hd_status hd_halo_chunks(const hd_mesh_desc *desc, int *nchunk, long long *chunk_units, long long *plan);

/* Number of kernels this library launched since the mesh was created (bench evidence). */
long long hd_launch_count(const hd_mesh *m);

const char *hd_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* HD_H */
