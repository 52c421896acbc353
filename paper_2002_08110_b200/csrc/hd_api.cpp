// hd_api.cpp -- the C ABI (include/hd.h): validation, mesh/partition plan, LSRK(5,4) driver.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <utility>

#include "hd_internal.h"

namespace {

thread_local char g_err[512] = "";

hd_status fail(hd_status st, const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return st;
}

hd_status cuda_fail(cudaError_t e, const char *what) {
  return fail(HD_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

// Carpenter-Kennedy five-stage fourth-order 2N-storage coefficients (reading C13, Williamson form
// S:507). Checked against the classical order conditions by tests/test_host.py.
const double kRkA[5] = {0.0, -567301805773.0 / 1357537059087.0, -2404267990393.0 / 2016746695238.0,
                        -3550918686646.0 / 2091501179385.0, -1275806237668.0 / 842570457699.0};
const double kRkB[5] = {1432997174477.0 / 9575080441755.0, 5161836677717.0 / 13612068292357.0,
                        1720146321549.0 / 2090206949498.0, 3134564353537.0 / 4481467310338.0,
                        2277821191437.0 / 14882151754819.0};

std::mutex g_tab_mu;
unsigned g_tab_uploaded[64];  // per device: bitmask of n whose tables are in constant memory

hd_status ensure_tables(hd_mesh *m) {
  std::lock_guard<std::mutex> lk(g_tab_mu);
  if (m->device < 0 || m->device >= 64) return fail(HD_ERR_ARG, "device id out of range");
  if (g_tab_uploaded[m->device] & (1u << m->n)) return HD_OK;
  cudaError_t e = hd::upload_tables(m->n, m->tab);
  if (e != cudaSuccess) return cuda_fail(e, "upload_tables");
  g_tab_uploaded[m->device] |= 1u << m->n;
  return HD_OK;
}

void fill_cell_params(hd_mesh *m, hd::CellParams &p) {
  std::memset(&p, 0, sizeof(p));
  const int d = m->d;
  const int C = m->geo.C;
  p.ncells = (int)m->ncells_local;
  p.nitems = (int)(m->ncells_local / C);
  p.jdet = m->jdet;
  if (const char *dbg = getenv("HD_DEBUG")) p.debug = atoi(dbg);
  int lstride = 1, istride = 1;
  for (int i = 0; i < d; ++i) {
    p.L[i] = (int)m->desc.cells[i];
    p.IL[i] = i == 0 ? p.L[0] / C : p.L[i];
    p.lstride[i] = lstride;
    p.istride[i] = istride;
    lstride *= p.L[i];
    istride *= p.IL[i];
    p.lo[i] = m->desc.lo[i];
    p.h[i] = m->h[i];
    p.inv_h[i] = 1.0 / m->h[i];
    p.a_const[i] = m->desc.a_const[i];
    for (int j = 0; j < d; ++j) p.a_lin[i][j] = m->desc.a_lin[6 * i + j];
    p.tmode[i] = m->tmode[i];
    p.dirneg[i] = m->tmode[i] != hd::kTraceNone ? m->dirneg[i] : 0;
    p.rmask[i] = m->rmask[i];
    p.tbuf[i] = m->tbuf[i];
  }
  p.flags = m->flags;
  // publication mask: phase ph (dims 2ph, 2ph+1) is published when one of its dims has traces
  // (consumers acquire it) or a ring dim of phase ph-1 checks it before overwriting a slot
  const int nph = m->geo.phases;
  for (int i = 0; i < d; ++i) {
    const int ph = i / 2;
    if (m->tmode[i] != hd::kTraceNone) p.pubmask |= 1 << ph;
    if (m->tmode[i] == hd::kTraceRing) p.pubmask |= 1 << (ph + 1);
  }
  (void)nph;
  // one epoch per cell-kernel launch; flags count warp publications cumulatively
  m->epoch += 1;
  p.target = (int)(m->epoch * m->geo.warps_per_item);
}

// Upwind-trace plan: a dim can use published traces when its speed
// sign depends only on slower dims (then the traversal can follow it); dims sorted by item stride
// get an L2-resident ring while the ring budget lasts, the rest a full-size buffer.
hd_status plan_traces(hd_mesh *m) {
  const int d = m->d;
  const hd::CellGeometry &g = m->geo;
  const long long fn = m->nd / m->n;  // face points
  int istride[6], IL0 = (int)(m->desc.cells[0] / g.C);
  long long st = 1;
  for (int i = 0; i < d; ++i) {
    istride[i] = (int)st;
    st *= i == 0 ? IL0 : m->desc.cells[i];
  }
  const long long nitems = m->ncells_local / g.C;
  double budget = 64.0 * (1 << 20);
  if (const char *e = getenv("HD_RING_MB")) budget = atof(e) * (1 << 20);
  bool use = true;
  if (const char *e = getenv("HD_TRACE")) use = atoi(e) != 0;
  int order[6];
  for (int i = 0; i < d; ++i) order[i] = i;
  for (int i = 0; i < d; ++i)
    for (int j = i + 1; j < d; ++j)
      if (istride[order[j]] < istride[order[i]]) std::swap(order[i], order[j]);
  double used = 0.0;
  for (int oi = 0; oi < d; ++oi) {
    const int i = order[oi];
    m->tmode[i] = hd::kTraceNone;
    m->rmask[i] = 0;
    m->tbuf[i] = nullptr;
    // eligible: the sign of a_i is the same on the whole box, so the traversal can follow it in
    // every cell with one global direction (then the producer of a cell's upwind trace is exactly
    // istride_i items earlier); a_i is affine, so check its extreme values at the box corners
    double amin = m->desc.a_const[i], amax = m->desc.a_const[i];
    for (int j = 0; j < d; ++j) {
      const double aj = m->desc.a_lin[6 * i + j];
      amin += fmin(aj * m->desc.lo[j], aj * m->desc.hi[j]);
      amax += fmax(aj * m->desc.lo[j], aj * m->desc.hi[j]);
    }
    m->dirneg[i] = amax <= 0.0 && amin < 0.0 ? 1 : 0;
    const bool eligible = use && m->desc.cells[i] > 1 && (amin >= 0.0 || amax <= 0.0);
    if (!eligible) continue;
    long long R = 1;
    while (R < (long long)istride[i] + 2LL * m->grid + 64) R <<= 1;
    const double ring_bytes = (double)R * g.C * fn * 8.0;
    size_t bytes;
    if (R < nitems && used + ring_bytes <= budget) {
      m->tmode[i] = hd::kTraceRing;
      m->rmask[i] = (int)(R - 1);
      used += ring_bytes;
      bytes = (size_t)ring_bytes;
    } else {
      m->tmode[i] = hd::kTraceFar;
      bytes = (size_t)nitems * g.C * fn * 8;
    }
    cudaError_t e = cudaMalloc(&m->tbuf[i], bytes);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(HD_ERR_OOM, "trace buffer of %zu bytes: %s", bytes, cudaGetErrorString(e));
    }
  }
  const size_t fbytes = (size_t)nitems * (g.phases + 1) * sizeof(int);
  cudaError_t e = cudaMalloc(&m->flags, fbytes);
  if (e == cudaSuccess) e = cudaMemset(m->flags, 0, fbytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(HD_ERR_OOM, "flag buffer: %s", cudaGetErrorString(e));
  }
  m->epoch = 0;
  return HD_OK;
}

void free_mesh(hd_mesh *m) {
  for (int i = 0; i < 6; ++i)
    if (m->tbuf[i]) cudaFree(m->tbuf[i]);
  if (m->flags) cudaFree(m->flags);
  delete m;
}

bool overlaps(const void *a, const void *b, size_t bytes) {
  const char *x = (const char *)a, *y = (const char *)b;
  return x < y + bytes && y < x + bytes;
}

}  // namespace

extern "C" {

const char *hd_last_error(void) { return g_err; }

hd_status hd_create_mesh(const hd_mesh_desc *desc, hd_mesh **out) {
  if (!desc || !out) return fail(HD_ERR_ARG, "null argument");
  *out = nullptr;
  const int d = desc->d_x + desc->d_v;
  if (desc->d_x < 1 || desc->d_x > 3 || desc->d_v < 1 || desc->d_v > 3)
    return fail(HD_ERR_ARG, "d_x, d_v must be in 1..3 (got %d, %d)", desc->d_x, desc->d_v);
  if (desc->k < 0) return fail(HD_ERR_ARG, "k must be >= 0");
  const int n = desc->k + 1;
  long long ncells = 1, cx_total = 1;
  for (int i = 0; i < d; ++i) {
    if (desc->cells[i] < 1) return fail(HD_ERR_ARG, "cells[%d] = %lld must be >= 1", i, desc->cells[i]);
    if (!(desc->hi[i] > desc->lo[i]) || !std::isfinite(desc->lo[i]) || !std::isfinite(desc->hi[i]))
      return fail(HD_ERR_ARG, "box of dim %d is empty or not finite", i);
    if (ncells > (1LL << 62) / desc->cells[i]) return fail(HD_ERR_ARG, "cell count overflows");
    ncells *= desc->cells[i];
    if (i < desc->d_x) cx_total *= desc->cells[i];
    if (desc->a_lin[6 * i + i] != 0.0) return fail(HD_ERR_ARG, "a_lin[%d][%d] must be 0 (divergence-free field)", i, i);
    if (!std::isfinite(desc->a_const[i])) return fail(HD_ERR_ARG, "a_const[%d] not finite", i);
  }
  for (int i = d; i < 6; ++i)
    for (int j = 0; j < 6; ++j)
      if (desc->a_lin[6 * i + j] != 0.0 || desc->a_lin[6 * j + i] != 0.0)
        return fail(HD_ERR_ARG, "a_lin entries beyond dimension d must be 0");
  long long nd = 1;
  for (int i = 0; i < d; ++i) nd *= n;
  if (n > 64 || ncells > (1LL << 62) / nd) return fail(HD_ERR_ARG, "DoF count overflows 64-bit indexing");
  if (desc->flux != 0) return fail(HD_ERR_UNSUPPORTED, "only the upwind flux (0) is built on the GPU path");
  if (n < 2 || n > 6 || !hd::cell_kernel_supported(d, n))
    return fail(HD_ERR_UNSUPPORTED, "(d=%d, n=%d) is not in the built kernel set", d, n);
  if (desc->nranks < 1 || desc->rank < 0 || desc->rank >= desc->nranks)
    return fail(HD_ERR_ARG, "rank %d / nranks %d invalid", desc->rank, desc->nranks);
  if (cx_total % desc->nranks != 0)
    return fail(HD_ERR_ARG, "nranks (%d) must divide |C_x| (%lld)", desc->nranks, cx_total);
  if (desc->nranks > 1) return fail(HD_ERR_UNSUPPORTED, "multi-rank halo not built yet");
  // the sign of each a_i must be constant on every cell (reading C11): check the affine field's
  // range over each 1D cell slab of the dims it depends on
  for (int i = 0; i < d; ++i) {
    bool any_lin = false;
    for (int j = 0; j < d; ++j) any_lin |= desc->a_lin[6 * i + j] != 0.0;
    if (!any_lin) continue;
    // enumerate all cells' ranges only along dims with a_lin != 0: the range over a cell is
    // a_const + sum_j [min,max] of a_lin[i][j] z_j over the cell's interval in dim j
    // (separable), so check the worst case combination per dim-product lazily via recursion.
    int dims[6], nd_ = 0;
    for (int j = 0; j < d; ++j)
      if (desc->a_lin[6 * i + j] != 0.0) dims[nd_++] = j;
    long long combos = 1;
    for (int t = 0; t < nd_; ++t) combos *= desc->cells[dims[t]];
    if (combos > 100000000LL) return fail(HD_ERR_UNSUPPORTED, "field sign check too large");
    for (long long cmb = 0; cmb < combos; ++cmb) {
      long long rr = cmb;
      double lo = desc->a_const[i], hi = desc->a_const[i];
      for (int t = 0; t < nd_; ++t) {
        const int j = dims[t];
        const long long c = rr % desc->cells[j];
        rr /= desc->cells[j];
        const double hj = (desc->hi[j] - desc->lo[j]) / (double)desc->cells[j];
        const double z0 = desc->lo[j] + c * hj, z1 = z0 + hj;
        const double aj = desc->a_lin[6 * i + j];
        lo += fmin(aj * z0, aj * z1);
        hi += fmax(aj * z0, aj * z1);
      }
      const double tol = 1e-12 * (fabs(lo) + fabs(hi) + 1.0);
      if (lo < -tol && hi > tol)
        return fail(HD_ERR_UNSUPPORTED, "sign of a_%d changes inside a cell (reading C11)", i);
    }
  }
  hd_mesh *m = new (std::nothrow) hd_mesh();
  if (!m) return fail(HD_ERR_OOM, "host allocation failed");
  m->desc = *desc;
  m->d = d;
  m->n = n;
  m->nd = nd;
  m->ncells_global = ncells;
  m->cx_total = cx_total;
  m->nx_local = cx_total / desc->nranks;
  m->cx_begin = m->nx_local * desc->rank;
  m->cx_end = m->cx_begin + m->nx_local;
  m->nv = ncells / cx_total;
  m->ncells_local = m->nx_local * m->nv;
  m->owned_dofs = m->ncells_local * nd;
  m->jdet = 1.0;
  for (int i = 0; i < d; ++i) {
    m->h[i] = (desc->hi[i] - desc->lo[i]) / (double)desc->cells[i];
    m->jdet *= m->h[i];
  }
  hd::build_tables(n, m->tab);
  cudaError_t e = cudaGetDevice(&m->device);
  if (e != cudaSuccess) {
    delete m;
    return cuda_fail(e, "cudaGetDevice");
  }
  e = cudaDeviceGetAttribute(&m->sms, cudaDevAttrMultiProcessorCount, m->device);
  if (e != cudaSuccess) {
    delete m;
    return cuda_fail(e, "cudaDeviceGetAttribute");
  }
  hd_status st = ensure_tables(m);
  if (st != HD_OK) {
    delete m;
    return st;
  }
  m->launches = 0;
  if (m->ncells_local >= (1LL << 31) || m->owned_dofs / m->n >= (1LL << 40)) {
    delete m;
    return fail(HD_ERR_UNSUPPORTED, "more than 2^31 cells per rank");
  }
  m->geo = hd::cell_geometry(d, n, (int)desc->cells[0]);
  e = hd::cell_grid_size(d, n, (int)desc->cells[0], 0, m->sms, &m->grid);
  if (e != cudaSuccess) {
    delete m;
    return cuda_fail(e, "cell kernel occupancy");
  }
  st = plan_traces(m);
  if (st != HD_OK) {
    free_mesh(m);
    return st;
  }
  *out = m;
  return HD_OK;
}

hd_status hd_destroy_mesh(hd_mesh *m) {
  if (!m) return fail(HD_ERR_ARG, "null mesh");
  free_mesh(m);
  return HD_OK;
}

hd_status hd_mesh_traces(const hd_mesh *m, int *tmode, int *ring_slots) {
  if (!m) return fail(HD_ERR_ARG, "null mesh");
  for (int i = 0; i < m->d; ++i) {
    if (tmode) tmode[i] = m->tmode[i];
    if (ring_slots) ring_slots[i] = m->tmode[i] == hd::kTraceRing ? m->rmask[i] + 1 : 0;
  }
  return HD_OK;
}

hd_status hd_mesh_info(const hd_mesh *m, long long *owned_dofs, long long *cx_begin, long long *cx_end) {
  if (!m) return fail(HD_ERR_ARG, "null mesh");
  if (owned_dofs) *owned_dofs = m->owned_dofs;
  if (cx_begin) *cx_begin = m->cx_begin;
  if (cx_end) *cx_end = m->cx_end;
  return HD_OK;
}

hd_status hd_tables_1d(int n, double *xi, double *w, double *K, double *lam, double *tau) {
  if (n < 2 || n > hd::kMaxN) return fail(HD_ERR_ARG, "n must be in 2..%d", hd::kMaxN);
  hd::Tables1D t;
  hd::build_tables(n, t);
  for (int i = 0; i < n; ++i) {
    if (xi) xi[i] = t.xi[i];
    if (w) w[i] = t.w[i];
  }
  for (int s = 0; s < 2; ++s)
    for (int i = 0; i < n; ++i) {
      if (lam) lam[s * n + i] = t.lam[s][i];
      if (tau) tau[s * n + i] = t.tau[s][i];
      for (int j = 0; j < n; ++j)
        if (K) K[(s * n + i) * n + j] = t.K[s][i][j];
    }
  return HD_OK;
}

hd_status hd_lsrk_coefficients(double *a, double *b) {
  if (!a || !b) return fail(HD_ERR_ARG, "null argument");
  for (int s = 0; s < 5; ++s) {
    a[s] = kRkA[s];
    b[s] = kRkB[s];
  }
  return HD_OK;
}

long long hd_launch_count(const hd_mesh *m) { return m ? m->launches : -1; }

hd_status hd_apply_advection(hd_mesh *m, const double *u, double *v, double t, void *stream) {
  (void)t;
  if (!m || !u || !v) return fail(HD_ERR_ARG, "null argument");
  if (overlaps(u, v, (size_t)m->owned_dofs * sizeof(double))) return fail(HD_ERR_ARG, "u and v overlap");
  hd_status st = ensure_tables(m);
  if (st != HD_OK) return st;
  hd::CellParams p;
  fill_cell_params(m, p);
  p.u = u;
  p.out = v;
  p.mode = hd::kModeAdvection;
  p.dtfac = 1.0;
  cudaError_t e = hd::launch_cell_kernel(m->d, m->n, p, (cudaStream_t)stream, &m->launches, m->grid);
  if (e != cudaSuccess) return cuda_fail(e, "advection kernel");
  return HD_OK;
}

static hd_status mass_impl(hd_mesh *m, double *u, void *stream, int inverse) {
  if (!m || !u) return fail(HD_ERR_ARG, "null argument");
  hd_status st = ensure_tables(m);
  if (st != HD_OK) return st;
  hd::StreamParams p;
  p.u = u;
  p.ndofs = m->owned_dofs;
  p.jdet = m->jdet;
  p.inverse = inverse;
  cudaError_t e = hd::launch_mass_kernel(m->d, m->n, p, (cudaStream_t)stream, &m->launches, m->sms);
  if (e != cudaSuccess) return cuda_fail(e, "mass kernel");
  return HD_OK;
}

hd_status hd_apply_inv_mass(hd_mesh *m, double *u, void *stream) { return mass_impl(m, u, stream, 1); }
hd_status hd_apply_mass(hd_mesh *m, double *u, void *stream) { return mass_impl(m, u, stream, 0); }

hd_status hd_rk_step(hd_mesh *m, double *buf[3], int *sol, double t, double dt, int nsteps, void *stream) {
  (void)t;
  if (!m || !buf || !sol) return fail(HD_ERR_ARG, "null argument");
  if (*sol < 0 || *sol > 2) return fail(HD_ERR_ARG, "*sol must be 0, 1 or 2");
  if (nsteps < 1) return fail(HD_ERR_ARG, "nsteps must be >= 1");
  if (!std::isfinite(dt)) return fail(HD_ERR_ARG, "dt not finite");
  const size_t bytes = (size_t)m->owned_dofs * sizeof(double);
  for (int i = 0; i < 3; ++i) {
    if (!buf[i]) return fail(HD_ERR_ARG, "null buffer %d", i);
    for (int j = 0; j < i; ++j)
      if (overlaps(buf[i], buf[j], bytes)) return fail(HD_ERR_ARG, "buffers %d and %d overlap", j, i);
  }
  hd_status st = ensure_tables(m);
  if (st != HD_OK) return st;
  hd::CellParams p;
  fill_cell_params(m, p);
  p.dtfac = dt;
  int iu = *sol, idu = (*sol + 1) % 3, iw = (*sol + 2) % 3;
  for (int step = 0; step < nsteps; ++step) {
    for (int s = 0; s < 5; ++s) {
      p.u = buf[iu];
      p.du = buf[idu];
      p.out = buf[iw];
      p.mode = s == 0 ? hd::kModeRKFirst : hd::kModeRK;
      p.rk_a = kRkA[s];
      p.rk_b = kRkB[s];
      // every launch is a new publication epoch for the trace flags
      if (step > 0 || s > 0) {
        m->epoch += 1;
        p.target = (int)(m->epoch * m->geo.warps_per_item);
      }
      cudaError_t e = hd::launch_cell_kernel(m->d, m->n, p, (cudaStream_t)stream, &m->launches, m->grid);
      if (e != cudaSuccess) return cuda_fail(e, "rk stage kernel");
      const int tmp = iu;
      iu = iw;
      iw = tmp;
    }
  }
  *sol = iu;
  return HD_OK;
}

hd_status hd_rk_step_host(hd_mesh *m, const double *u_host, double *u_out_host, double *dbuf[3], double t, double dt,
                          int nsteps, void *stream) {
  if (!m || !u_host || !u_out_host || !dbuf) return fail(HD_ERR_ARG, "null argument");
  const size_t bytes = (size_t)m->owned_dofs * sizeof(double);
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaMemcpyAsync(dbuf[0], u_host, bytes, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return cuda_fail(e, "H2D copy");
  int sol = 0;
  hd_status st = hd_rk_step(m, dbuf, &sol, t, dt, nsteps, stream);
  if (st != HD_OK) return st;
  e = cudaMemcpyAsync(u_out_host, dbuf[sol], bytes, cudaMemcpyDeviceToHost, s);
  if (e != cudaSuccess) return cuda_fail(e, "D2H copy");
  e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "stream synchronize");
  return HD_OK;
}

hd_status hd_fill_initial(hd_mesh *m, double *u, int recipe, unsigned long long seed, void *stream) {
  if (!m || !u) return fail(HD_ERR_ARG, "null argument");
  if (recipe < 0 || recipe > 3) return fail(HD_ERR_ARG, "recipe must be 0..3");
  if (recipe == 0 && m->d < 2) return fail(HD_ERR_ARG, "gauss2d needs d >= 2");
  hd_status st = ensure_tables(m);
  if (st != HD_OK) return st;
  hd::FillParams p;
  std::memset(&p, 0, sizeof(p));
  p.u = u;
  p.ncells = m->ncells_local;
  p.nx_local = m->nx_local;
  p.cx_begin = m->cx_begin;
  for (int i = 0; i < m->d; ++i) {
    p.L[i] = m->desc.cells[i];
    p.lo[i] = m->desc.lo[i];
    p.h[i] = m->h[i];
  }
  p.d_x = m->desc.d_x;
  p.d = m->d;
  p.recipe = recipe;
  p.seed = seed;
  cudaError_t e = hd::launch_fill_kernel(m->d, m->n, p, (cudaStream_t)stream, &m->launches);
  if (e != cudaSuccess) return cuda_fail(e, "fill kernel");
  return HD_OK;
}

}  // extern "C"
