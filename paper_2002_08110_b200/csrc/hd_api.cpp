// hd_api.cpp -- the C ABI (include/hd.h): validation, mesh/partition plan, LSRK(5,4) driver.
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <utility>
#include <vector>

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
// S:507). Checked against the classical order conditions by tests/test_abi.py and tests/test_oracle_lsrk.py.
const double kRkA[5] = {0.0, -567301805773.0 / 1357537059087.0, -2404267990393.0 / 2016746695238.0,
                        -3550918686646.0 / 2091501179385.0, -1275806237668.0 / 842570457699.0};
const double kRkB[5] = {1432997174477.0 / 9575080441755.0, 5161836677717.0 / 13612068292357.0,
                        1720146321549.0 / 2090206949498.0, 3134564353537.0 / 4481467310338.0,
                        2277821191437.0 / 14882151754819.0};

// ---- NCCL, loaded at run time (only multi-rank meshes with a ncclUniqueId need it; torch's NCCL is
// picked up when it is already loaded). Minimal prototypes of the stable NCCL C API.
typedef struct {
  char internal[128];
} nccl_unique_id;
typedef int nccl_result;
constexpr int kNcclFloat64 = 8;
constexpr int kNcclInt32 = 2;

}  // namespace

namespace hd {
struct NcclApi {
  bool ok = false;
  nccl_result (*get_unique_id)(nccl_unique_id *) = nullptr;
  nccl_result (*comm_init_rank)(void **, int, nccl_unique_id, int) = nullptr;
  nccl_result (*comm_destroy)(void *) = nullptr;
  nccl_result (*send)(const void *, size_t, int, int, void *, cudaStream_t) = nullptr;
  nccl_result (*recv)(void *, size_t, int, int, void *, cudaStream_t) = nullptr;
  nccl_result (*group_start)() = nullptr;
  nccl_result (*group_end)() = nullptr;
  const char *(*error_string)(nccl_result) = nullptr;
};
}  // namespace hd

namespace {

hd::NcclApi g_nccl;
std::mutex g_nccl_mu;

hd_status load_nccl() {
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  if (g_nccl.ok) return HD_OK;
  void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return fail(HD_ERR_NCCL, "cannot load libnccl.so.2: %s", dlerror());
#define HD_SYM(field, name)                                                        \
  *(void **)(&g_nccl.field) = dlsym(h, name);                                      \
  if (!g_nccl.field) return fail(HD_ERR_NCCL, "libnccl.so.2 lacks %s", name);
  HD_SYM(get_unique_id, "ncclGetUniqueId")
  HD_SYM(comm_init_rank, "ncclCommInitRank")
  HD_SYM(comm_destroy, "ncclCommDestroy")
  HD_SYM(send, "ncclSend")
  HD_SYM(recv, "ncclRecv")
  HD_SYM(group_start, "ncclGroupStart")
  HD_SYM(group_end, "ncclGroupEnd")
  HD_SYM(error_string, "ncclGetErrorString")
#undef HD_SYM
  g_nccl.ok = true;
  return HD_OK;
}

hd_status nccl_fail(nccl_result r, const char *what) {
  return fail(HD_ERR_NCCL, "%s: %s", what, g_nccl.error_string ? g_nccl.error_string(r) : "?");
}

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

// Kernel parameters of a mesh (the launch-dependent fields -- vectors, mode, stage coefficients, epoch --
// are set by launch_stage).
void fill_cell_params(hd_mesh *m, hd::CellParams &p) {
  std::memset(&p, 0, sizeof(p));
  const int d = m->d, n = m->n;
  const hd::CellGeometry &g = m->geo;
  p.CT = g.CT;
  p.GPU = g.GPU * m->slab;
  p.slab = m->slab;
  p.FN = (int)(m->nd / m->n);
  p.ND = (int)m->nd;
  p.prefetch = (m->nd * 8) % 16 == 0 ? 1 : 0;
  p.nunits = m->nunits / m->slab;
  p.jdet = m->jdet;
  p.cstride = g.pencil ? m->pt.len[0] : 1;
  p.sched = m->sched;
  p.schedc = m->schedc;
  p.flags = m->flags;
  p.uctr = m->dbg + 32;
  p.dtfac = 1.0;
  p.err = m->dbg;
  p.stag = m->dbg + 1;
  p.rtag = m->dbg + 13;
  p.ncells = m->ncells_local;
  for (int i = 0; i < 6; ++i) p.nhalo[i] = m->halo[i].n_from_left + m->halo[i].n_from_right;
  for (int i = 0; i < d; ++i) {
    p.L[i] = (int)m->pt.len[i];
    p.coff[i] = (int)m->pt.off[i];
    if (m->pt.parts[i] > 1) p.hbuf[i] = m->hbuf[i];
    p.lo[i] = m->desc.lo[i];
    p.h[i] = m->h[i];
    p.inv_h[i] = 1.0 / m->h[i];
    p.a_const[i] = m->desc.a_const[i];
    bool var = false;
    for (int j = 0; j < d; ++j) {
      p.a_lin[i][j] = m->desc.a_lin[6 * i + j];
      var = var || p.a_lin[i][j] != 0.0;
    }
    p.var[i] = var ? 1 : 0;
    p.tbuf[i] = m->tbuf[i];
  }
  (void)n;
}

// The speed-prescaled tables of the constant-speed dims for a launch with time factor dtfac (1 for A,
// dt for an RK stage): s_i K[s], s_i tau[s], s_i = a_i dtfac / h_i, compact [dim][sign][N][N] / [N]. The
// line speed is formed exactly as the kernel's line_speed does for a constant field ((a_i + 0) * fac).
void set_dtfac(hd_mesh *m, hd::CellParams &p, double dtfac) {
  // central flux: each of the two one-sided operators enters with weight 1/2
  if (m->desc.flux == 1) dtfac *= 0.5;
  p.dtfac = dtfac;
  const int N = m->n;
  for (int i = 0; i < m->d; ++i) {
    p.fac[i] = dtfac * p.inv_h[i];
    for (int j = 0; j < m->d; ++j) p.slin[i][j] = p.a_lin[i][j] * p.h[j] * p.fac[i];
  }
  for (int i = 0; i < m->d; ++i) {
    const double si = p.var[i] ? 1.0 : (p.a_const[i] + 0.0) * (dtfac * p.inv_h[i]);
    for (int sg = 0; sg < 2; ++sg) {
      for (int a = 0; a < N; ++a) {
        for (int j = 0; j < N; ++j) p.Ks[((i * 2 + sg) * N + a) * N + j] = si * m->tab.K[sg][a][j];
        p.Ts[(i * 2 + sg) * N + a] = si * m->tab.tau[sg][a];
      }
    }
  }
}

// Every cell-kernel launch is a new epoch; unit flags hold (epoch << 10) | steps done. Before the epoch
// field overflows, the flags are cleared on the launch stream (ordered after every earlier launch on it)
// and the count restarts.
hd_status next_epoch(hd_mesh *m, hd::CellParams &p, cudaStream_t s) {
  m->epoch += 1;
  if (m->epoch >= (1LL << 20)) {
    if (m->flags) {
      cudaError_t e = cudaMemsetAsync(m->flags, 0, (size_t)m->nflags * sizeof(int), s);
      if (e != cudaSuccess) return cuda_fail(e, "flag reset");
    }
    m->epoch = 1;
  }
  p.epoch = (int)(m->epoch << 10);
  return HD_OK;
}

void free_mesh(hd_mesh *m) {
  for (int i = 0; i < 6; ++i)
    if (m->tbuf[i]) cudaFree(m->tbuf[i]);
  if (m->flags) cudaFree(m->flags);
  if (m->sched) cudaFree(m->sched);
  if (m->sched2) cudaFree(m->sched2);
  if (m->schedc2) cudaFree(m->schedc2);
  if (m->dbg) cudaFree(m->dbg);
  if (m->schedc) cudaFree(m->schedc);
  for (int i = 0; i < 6; ++i) {
    if (m->hbuf[i]) cudaFree(m->hbuf[i]);
    if (m->hslot[i]) cudaFree(m->hslot[i]);
  }
  if (m->pack_cells) cudaFree(m->pack_cells);
  if (m->pack_dimsg) cudaFree(m->pack_dimsg);
  if (m->sendbuf) cudaFree(m->sendbuf);
  if (m->fcl_tr) cudaFree(m->fcl_tr);
  if (m->fcl_G) cudaFree(m->fcl_G);
  if (m->vp_rho) cudaFree(m->vp_rho);
  if (m->vp_rhohat) cudaFree(m->vp_rhohat);
  if (m->vp_E) cudaFree(m->vp_E);
  if (m->nccl_comm && g_nccl.ok) g_nccl.comm_destroy(m->nccl_comm);
  for (int c = 0; c < hd::kMaxChunk; ++c)
    if (m->ev_chunk[c]) cudaEventDestroy(m->ev_chunk[c]);
  if (m->ev_u) cudaEventDestroy(m->ev_u);
  if (m->comm) cudaStreamDestroy(m->comm);
  delete m;
}

template <class T>
hd_status upload(T **dst, const T *src, size_t count, const char *what) {
  *dst = nullptr;
  if (count == 0) return HD_OK;
  cudaError_t e = cudaMalloc(dst, count * sizeof(T));
  if (e == cudaSuccess && src) e = cudaMemcpy(*dst, src, count * sizeof(T), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(HD_ERR_OOM, "%s (%zu bytes): %s", what, count * sizeof(T), cudaGetErrorString(e));
  }
  return HD_OK;
}

// Upwind-trace plan (DESIGN.md §6 "Upwind traces"). In pencil mode a dim i >= 1 FOLLOWS its speed when a_i
// depends on slower dims only (its sign is then constant along the traversal of dim i and of all faster
// dims, so the sweep can go upwind -> downwind); every following dim publishes its downwind traces for
// the neighbour one group later.
hd_status plan_traces(hd_mesh *m) {
  const int d = m->d;
  const hd::CellGeometry &g = m->geo;
  const long long fn = m->nd / m->n;  // face points
  const bool use = g.pencil && g.GPU <= 1023;
  bool any = false;
  for (int i = 0; i < d; ++i) {
    m->pub[i] = 0;
    m->follow[i] = 0;
    m->tbuf[i] = nullptr;
    if (i == 0 || !g.pencil || m->pt.len[i] < 2) continue;
    bool follow = true;  // (central flux: the forced sides are constant, every dim follows)
    for (int j = 0; j < i && m->desc.flux == 0; ++j) follow = follow && m->desc.a_lin[6 * i + j] == 0.0;
    m->follow[i] = follow ? 1 : 0;
    if (!follow || !use) continue;
    m->pub[i] = 1;
    const size_t bytes = (size_t)m->ncells_local * fn * sizeof(double);
    cudaError_t e = cudaMalloc(&m->tbuf[i], bytes);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(HD_ERR_OOM, "trace buffer of %zu bytes: %s", bytes, cudaGetErrorString(e));
    }
    any = true;
  }
  m->flags = nullptr;
  m->nflags = 0;
  if (any) {
    // rounded up to whole 16-byte words
    m->nflags = ((long long)m->nunits + 3) / 4 * 4;
    const size_t fbytes = (size_t)m->nflags * sizeof(int);
    cudaError_t e = cudaMalloc(&m->flags, fbytes);
    if (e == cudaSuccess) e = cudaMemset(m->flags, 0, fbytes);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(HD_ERR_OOM, "flag buffer: %s", cudaGetErrorString(e));
    }
  }
  m->epoch = 0;
  // skew (steps a same-round producer runs ahead of its consumer): 2 gives the producer a full step of
  // margin; the first `skew` steps of a pencil then read their upwind neighbours directly
#ifndef HD_SLAB
#define HD_SLAB 0
#endif
#ifndef HD_SKEW
#define HD_SKEW 2
#endif
  m->skew = g.pencil && g.GPU > HD_SKEW ? HD_SKEW : (g.pencil && g.GPU > 1 ? 1 : 0);
  return HD_OK;
}

// Build the static schedule of the cell kernel (hd_sched.cpp) and upload it (after the halo plan: halo
// sources carry receive-buffer slots).
hd_status upload_schedule(hd_mesh *m) {
  std::vector<hd::SchedDim> recs;
  std::vector<hd::SchedCell> cells;
  const bool central = m->desc.flux == 1;
  hd::build_schedule(*m, recs, cells, central ? 0 : -1);
  hd_status st = upload(&m->sched, recs.data(), recs.size(), "schedule");
  if (st == HD_OK) st = upload(&m->schedc, cells.data(), cells.size(), "schedule");
  if (st == HD_OK && central) {
    hd::build_schedule(*m, recs, cells, 1);
    st = upload(&m->sched2, recs.data(), recs.size(), "schedule");
    if (st == HD_OK) st = upload(&m->schedc2, cells.data(), cells.size(), "schedule");
  }
  return st;
}

// Halo plan and buffers of a multi-rank mesh (hd_plan.cpp), cut into v-chunks: in pencil mode
// the units are ordered with the slowest dim (a v dim, never split) outermost, so a range of its
// traversal coordinate is a contiguous unit range, and -- the halo plane order also having that dim
// slowest -- a contiguous range of every send list and receive buffer.
// The v-chunk plan of a multi-rank mesh, host only (also behind the hd_halo_chunks query): chunk unit ranges
// and, per chunk and x dim, the (offset, count) of the send-list entries to the right / left rank and of the
// receive slots from the left / right rank; the chunk-major send list itself (cells, dim | sign << 8).
struct ChunkPlan {
  int nchunk = 1;
  int chunk_u[hd::kMaxChunk + 1] = {};
  hd_mesh::ChunkHalo chunk[hd::kMaxChunk] = {};
  std::vector<int> cells, dimsg;
};
void build_chunk_plan(const hd_mesh_desc &ds, const hd::Partition &pt, const double *h, const hd::CellGeometry &geo,
                      long long nunits, bool follow_last, const hd::HaloDim *halo, ChunkPlan &cp) {
  const int d = pt.d;
  const long long Ls = pt.len[d - 1];
  cp = ChunkPlan();
  // chunks are ranges of the slowest dim, which must then not be split itself (its halo would cross chunks)
  cp.nchunk = geo.pencil && pt.parts[d - 1] == 1 ? (int)std::min<long long>(4, Ls) : 1;
  bool reversed = false;
  if (geo.pencil && follow_last) {
    long long cg[6];
    for (int j = 0; j < d; ++j) cg[j] = pt.off[j];
    reversed = hd::host_cell_sign(ds, h, d, d - 1, cg) != 0;
  }
  long long tcut[hd::kMaxChunk + 1];
  for (int c = 0; c <= cp.nchunk; ++c) tcut[c] = c * Ls / cp.nchunk;
  const long long units_per_slice = cp.nchunk > 1 ? nunits / Ls : 0;
  for (int c = 0; c <= cp.nchunk; ++c)
    cp.chunk_u[c] = cp.nchunk > 1 ? (int)(tcut[c] * units_per_slice) : (c ? (int)nunits : 0);
  for (int c = 0; c < cp.nchunk; ++c) {
    hd_mesh::ChunkHalo &ch = cp.chunk[c];
    ch.pe0 = (long long)cp.cells.size();
    long long c0 = 0, c1 = Ls;  // cell range of the slowest coordinate
    if (cp.nchunk > 1) {
      c0 = reversed ? Ls - tcut[c + 1] : tcut[c];
      c1 = reversed ? Ls - tcut[c] : tcut[c + 1];
    }
    for (int i = 0; i < d; ++i) {
      const hd::HaloDim &hd = halo[i];
      if (!hd.active) continue;
      // plane positions of the chunk: [j0, j1) (the slowest dim is slowest in the plane order too)
      const long long plane = (long long)hd.slot.size(), per = plane / Ls;
      const long long j0 = c0 * per, j1 = c1 * per;
      long long before0 = 0, before1 = 0, in0 = 0, in1 = 0;  // sign-0 / sign-1 positions before / in [j0, j1)
      for (long long j = 0; j < j1; ++j) {
        const bool s1 = hd.slot[j] >= hd.n_from_left;
        if (j < j0) (s1 ? before1 : before0) += 1;
        else (s1 ? in1 : in0) += 1;
      }
      // to the right rank: my high-face cells with a_i > 0 (sign 0), in plane order; to the left: sign 1
      ch.sr[i][0] = (long long)cp.cells.size();
      ch.sr[i][1] = in0;
      for (long long q = before0; q < before0 + in0; ++q) {
        cp.cells.push_back(hd.send_right[q]);
        cp.dimsg.push_back(i);
      }
      ch.sl[i][0] = (long long)cp.cells.size();
      ch.sl[i][1] = in1;
      for (long long q = before1; q < before1 + in1; ++q) {
        cp.cells.push_back(hd.send_left[q]);
        cp.dimsg.push_back(i | (1 << 8));
      }
      ch.rl[i][0] = before0;
      ch.rl[i][1] = in0;
      ch.rr[i][0] = hd.n_from_left + before1;
      ch.rr[i][1] = in1;
      ch.srq[i] = before0;
      ch.slq[i] = before1;
    }
    ch.pe1 = (long long)cp.cells.size();
  }
}

// Halo plan and buffers of a multi-rank mesh (hd_plan.cpp), cut into v-chunks: in pencil mode
// the units are ordered with the slowest dim (a v dim, never split) outermost, so a range of its
// traversal coordinate is a contiguous unit range, and -- the halo plane order also having that dim
// slowest -- a contiguous range of every send list and receive buffer.
hd_status setup_halo(hd_mesh *m) {
  const long long fn = m->nd / m->n;
  for (int i = 0; i < m->d; ++i) hd::make_halo(m->desc, m->pt, m->h, i, m->halo[i]);
  ChunkPlan cp;
  build_chunk_plan(m->desc, m->pt, m->h, m->geo, m->nunits, m->follow[m->d - 1] != 0, m->halo, cp);
  m->nchunk = cp.nchunk;
  std::memcpy(m->chunk_u, cp.chunk_u, sizeof(m->chunk_u));
  std::memcpy(m->chunk, cp.chunk, sizeof(m->chunk));
  for (int i = 0; i < m->d; ++i) {
    const hd::HaloDim &hd = m->halo[i];
    if (!hd.active) continue;
    hd_status st = upload(&m->hslot[i], hd.slot.data(), hd.slot.size(), "halo slot table");
    if (st != HD_OK) return st;
    st = upload(&m->hbuf[i], (const double *)nullptr, (size_t)(hd.n_from_left + hd.n_from_right) * fn,
                "halo receive buffer");
    if (st != HD_OK) return st;
  }
  m->nsend = (long long)cp.cells.size();
  hd_status st = upload(&m->pack_cells, cp.cells.data(), cp.cells.size(), "halo pack list");
  if (st == HD_OK) st = upload(&m->pack_dimsg, cp.dimsg.data(), cp.dimsg.size(), "halo pack list");
  if (st == HD_OK) st = upload(&m->sendbuf, (const double *)nullptr, (size_t)m->nsend * fn, "halo send buffer");
  return st;
}

// Pack the outgoing traces of chunk c of u (every stage: the operator input changes) with the launch's
// speeds, into the chunk's part of the send buffer.
hd_status halo_pack(hd_mesh *m, const hd::CellParams &p, const double *u, int c, cudaStream_t s) {
  const hd_mesh::ChunkHalo &ch = m->chunk[c];
  if (ch.pe1 == ch.pe0) return HD_OK;
  const long long fn = m->nd / m->n;
  hd::PackParams pp;
  pp.u = u;
  pp.out = m->sendbuf + ch.pe0 * fn;
  pp.cells = m->pack_cells + ch.pe0;
  pp.dimsg = m->pack_dimsg + ch.pe0;
  pp.nent = ch.pe1 - ch.pe0;
  cudaError_t e = hd::launch_pack_kernel(m->d, m->n, pp, p, s, &m->launches);
  if (e != cudaSuccess) return cuda_fail(e, "halo pack kernel");
  return HD_OK;
}

// NCCL transport, chunk c: one group; per peer the order is canonical on both sides (dims ascending; per
// dim: send to the right before send to the left, receive from the left before receive from the right),
// so every send meets its receive even when left == right (two ranks along a dim). Both sides compute the
// same counts (v is never split), so the zero-count skips agree.
hd_status halo_exchange_nccl(hd_mesh *m, int c, cudaStream_t s) {
  const long long fn = m->nd / m->n;
  const hd_mesh::ChunkHalo &ch = m->chunk[c];
  nccl_result r = g_nccl.group_start();
  if (r) return nccl_fail(r, "ncclGroupStart");
  for (int i = 0; i < m->d; ++i) {
    const hd::HaloDim &hd = m->halo[i];
    if (!hd.active) continue;
    if (ch.sr[i][1]) r = g_nccl.send(m->sendbuf + ch.sr[i][0] * fn, ch.sr[i][1] * fn, kNcclFloat64, hd.right, m->nccl_comm, s);
    if (!r && ch.sl[i][1])
      r = g_nccl.send(m->sendbuf + ch.sl[i][0] * fn, ch.sl[i][1] * fn, kNcclFloat64, hd.left, m->nccl_comm, s);
    if (!r && ch.rl[i][1])
      r = g_nccl.recv(m->hbuf[i] + ch.rl[i][0] * fn, ch.rl[i][1] * fn, kNcclFloat64, hd.left, m->nccl_comm, s);
    if (!r && ch.rr[i][1])
      r = g_nccl.recv(m->hbuf[i] + ch.rr[i][0] * fn, ch.rr[i][1] * fn, kNcclFloat64, hd.right, m->nccl_comm, s);
#ifdef HD_DEBUG
    // freshness tags travel with the traces; every rank runs the same build
    if (!r) r = g_nccl.send(m->dbg + 1 + i * 2, 1, kNcclInt32, hd.right, m->nccl_comm, s);
    if (!r) r = g_nccl.send(m->dbg + 2 + i * 2, 1, kNcclInt32, hd.left, m->nccl_comm, s);
    if (!r) r = g_nccl.recv(m->dbg + 13 + i * 2, 1, kNcclInt32, hd.left, m->nccl_comm, s);
    if (!r) r = g_nccl.recv(m->dbg + 14 + i * 2, 1, kNcclInt32, hd.right, m->nccl_comm, s);
#endif
    if (r) {
      g_nccl.group_end();
      return nccl_fail(r, "ncclSend/ncclRecv");
    }
  }
  r = g_nccl.group_end();
  if (r) return nccl_fail(r, "ncclGroupEnd");
  return HD_OK;
}

// Loopback transport, chunk c (all ranks' meshes in this process on one device): device copies from each
// neighbour's send buffer into the receive buffer, in the layout NCCL would deliver.
hd_status halo_exchange_loopback(hd_mesh **ms, int P, int c, cudaStream_t s) {
  for (int r = 0; r < P; ++r) {
    hd_mesh *m = ms[r];
    const long long fn = m->nd / m->n;
    const hd_mesh::ChunkHalo &ch = m->chunk[c];
    for (int i = 0; i < m->d; ++i) {
      const hd::HaloDim &hd = m->halo[i];
      if (!hd.active) continue;
      const hd_mesh *L = ms[hd.left], *R = ms[hd.right];
      cudaError_t e = cudaSuccess;
      if (ch.rl[i][1])
        e = cudaMemcpyAsync(m->hbuf[i] + ch.rl[i][0] * fn, L->sendbuf + L->chunk[c].sr[i][0] * fn,
                            ch.rl[i][1] * fn * sizeof(double), cudaMemcpyDeviceToDevice, s);
      if (e == cudaSuccess && ch.rr[i][1])
        e = cudaMemcpyAsync(m->hbuf[i] + ch.rr[i][0] * fn, R->sendbuf + R->chunk[c].sl[i][0] * fn,
                            ch.rr[i][1] * fn * sizeof(double), cudaMemcpyDeviceToDevice, s);
#ifdef HD_DEBUG
      // freshness tags travel with the traces
      if (e == cudaSuccess) e = cudaMemcpyAsync(m->dbg + 13 + i * 2, L->dbg + 1 + i * 2, sizeof(int), cudaMemcpyDeviceToDevice, s);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(m->dbg + 14 + i * 2, R->dbg + 2 + i * 2, sizeof(int), cudaMemcpyDeviceToDevice, s);
#endif
      if (e != cudaSuccess) return cuda_fail(e, "loopback halo copy");
    }
  }
  return HD_OK;
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
  if (desc->flux != 0 && desc->flux != 1) return fail(HD_ERR_ARG, "flux must be 0 (upwind) or 1 (central)");
  if (desc->flux == 1 && desc->nranks > 1)
    return fail(HD_ERR_UNSUPPORTED, "the central flux is built for single-rank meshes only");
  if (n < 2 || n > 6 || !hd::cell_kernel_supported(d, n))
    return fail(HD_ERR_UNSUPPORTED, "(d=%d, n=%d) is not in the built kernel set", d, n);
  if (desc->nranks < 1 || desc->rank < 0 || desc->rank >= desc->nranks)
    return fail(HD_ERR_ARG, "rank %d / nranks %d invalid", desc->rank, desc->nranks);
  hd::Partition pt;
  {
    std::string err;
    if (!hd::make_partition(*desc, pt, err)) return fail(HD_ERR_ARG, "%s", err.c_str());
  }
  // the sign of each a_i must be constant on every cell (reading C11): check the affine field's
  // range over each 1D cell slab of the dims it depends on
  for (int i = 0; i < d && desc->flux == 0; ++i) {  // (the central flux never selects a side)
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
  m->pt = pt;
  m->ncells_global = ncells;
  m->cx_total = cx_total;
  m->ncells_local = pt.ncells_local;
  m->owned_dofs = m->ncells_local * nd;
  {
    // flat x-cell range of the local box when it is contiguous (x-slab or one rank), else -1
    long long lo = 0, st = 1, cnt = 1;
    for (int i = 0; i < desc->d_x; ++i) {
      lo += pt.off[i] * st;
      st *= desc->cells[i];
      cnt *= pt.len[i];
    }
    bool contiguous = true;
    for (int i = 0; i + 1 < desc->d_x; ++i)
      if (pt.parts[i] > 1) contiguous = false;
    for (int i = desc->d_x; i < d; ++i)
      if (pt.parts[i] > 1) contiguous = false;
    m->cx_begin = contiguous ? lo : -1;
    m->cx_end = contiguous ? lo + cnt : -1;
  }
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
  if (m->ncells_local >= (1LL << 31)) {
    delete m;
    return fail(HD_ERR_UNSUPPORTED, "more than 2^31 cells per rank");
  }
  {
    // pencil mode needs one dim-0 direction per group: a_0 must not depend on z_1
    const int pencil_ok = d < 2 || m->desc.a_lin[6 * 0 + 1] == 0.0 || m->desc.flux == 1;
    m->geo = hd::cell_geometry(d, n, (int)pt.len[0], (int)pt.len[1], m->ncells_local, pencil_ok);
  }
  m->nunits = (int)(m->geo.pencil ? m->ncells_local / (pt.len[0] * m->geo.CT) : m->ncells_local / m->geo.CT);
  m->slab = 1;
  e = hd::cell_grid_size(d, n, m->geo, m->sms, &m->grid);
  if (e != cudaSuccess) {
    delete m;
    return cuda_fail(e, "cell kernel occupancy");
  }
  st = plan_traces(m);
  if (st == HD_OK) {
    // [0..31] debug words (HD_DEBUG), [32] the unit counter of the cell kernel
    cudaError_t e2 = cudaMalloc(&m->dbg, 64 * sizeof(int));
    if (e2 == cudaSuccess) e2 = cudaMemset(m->dbg, 0, 64 * sizeof(int));
    if (e2 != cudaSuccess) st = cuda_fail(e2, "debug words");
  }
  m->nchunk = 1;
  m->chunk_u[0] = 0;
  m->chunk_u[1] = m->nunits;
  std::memset(m->chunk, 0, sizeof(m->chunk));
  if (st == HD_OK && desc->nranks > 1) st = setup_halo(m);
  if (st == HD_OK && desc->nranks > 1 && desc->nccl_id) {
    cudaError_t e2 = cudaStreamCreateWithFlags(&m->comm, cudaStreamNonBlocking);
    if (e2 == cudaSuccess) e2 = cudaEventCreateWithFlags(&m->ev_u, cudaEventDisableTiming);
    for (int c = 0; c < m->nchunk && e2 == cudaSuccess; ++c)
      e2 = cudaEventCreateWithFlags(&m->ev_chunk[c], cudaEventDisableTiming);
    if (e2 != cudaSuccess) st = cuda_fail(e2, "halo stream / events");
  }
  if (st == HD_OK) {
    // slab super-units (one-chunk pencil meshes whose dim 1 publishes and is traversed upwind first): the
    // dim-1 traces then stay inside one CTA, one row of the slab apart -- kept in L2.
    // Off by default (HD_SLAB=1 builds it): 6% less DRAM traffic per 6D stage, but 1.4% slower (6D) and 5%
    // slower (5D: small wavefront hyperplanes of slabs put producers in their consumers' round)
    const int R = m->geo.pencil ? (int)(m->pt.len[1] / m->geo.CT) : 1;
    m->slab = (HD_SLAB && m->nchunk == 1 && R > 1 && m->pub[1] && m->follow[1] && (long long)R * m->geo.GPU < 1000) ? R : 1;
    if (m->nchunk == 1) m->chunk_u[1] = m->nunits / m->slab;
    st = upload_schedule(m);
  }
  if (st == HD_OK && desc->nranks > 1 && desc->nccl_id) {
    st = load_nccl();
    if (st == HD_OK) {
      nccl_unique_id id;
      std::memcpy(&id, desc->nccl_id, sizeof(id));
      nccl_result r = g_nccl.comm_init_rank(&m->nccl_comm, desc->nranks, id, desc->rank);
      if (r) {
        m->nccl_comm = nullptr;
        st = nccl_fail(r, "ncclCommInitRank");
      }
    }
  }
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
    if (tmode) tmode[i] = m->pub[i] ? 2 : 0;
    if (ring_slots) ring_slots[i] = 0;
  }
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

static hd_status mass_impl(hd_mesh *m, double *u, void *stream, int inverse) {
  if (!m || !u) return fail(HD_ERR_ARG, "null argument");
  if (reinterpret_cast<uintptr_t>(u) % 16 != 0) return fail(HD_ERR_ARG, "u is not 16-byte aligned");
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

long long hd_launch_count(const hd_mesh *m) { return m ? m->launches : -1; }

hd_status hd_apply_inv_mass(hd_mesh *m, double *u, void *stream) { return mass_impl(m, u, stream, 1); }
hd_status hd_apply_mass(hd_mesh *m, double *u, void *stream) { return mass_impl(m, u, stream, 0); }

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

hd_status hd_mesh_info(const hd_mesh *m, long long *owned_dofs, long long *cx_begin, long long *cx_end) {
  if (!m) return fail(HD_ERR_ARG, "null mesh");
  if (owned_dofs) *owned_dofs = m->owned_dofs;
  if (cx_begin) *cx_begin = m->cx_begin;
  if (cx_end) *cx_end = m->cx_end;
  return HD_OK;
}

hd_status hd_mesh_box(const hd_mesh *m, long long *off, long long *len, int *xparts) {
  if (!m) return fail(HD_ERR_ARG, "null mesh");
  for (int i = 0; i < 6; ++i) {
    if (off) off[i] = i < m->d ? m->pt.off[i] : 0;
    if (len) len[i] = i < m->d ? m->pt.len[i] : 1;
  }
  for (int i = 0; i < 3; ++i)
    if (xparts) xparts[i] = i < m->desc.d_x ? m->pt.parts[i] : 1;
  return HD_OK;
}

hd_status hd_nccl_unique_id(void *out) {
  if (!out) return fail(HD_ERR_ARG, "null argument");
  hd_status st = load_nccl();
  if (st != HD_OK) return st;
  nccl_unique_id id;
  nccl_result r = g_nccl.get_unique_id(&id);
  if (r) return nccl_fail(r, "ncclGetUniqueId");
  std::memcpy(out, &id, sizeof(id));
  return HD_OK;
}

hd_status hd_partition_info(const hd_mesh_desc *desc, int *xparts, long long *off, long long *len) {
  if (!desc) return fail(HD_ERR_ARG, "null argument");
  if (desc->nranks < 1 || desc->rank < 0 || desc->rank >= desc->nranks)
    return fail(HD_ERR_ARG, "rank %d / nranks %d invalid", desc->rank, desc->nranks);
  hd::Partition pt;
  std::string err;
  if (!hd::make_partition(*desc, pt, err)) return fail(HD_ERR_ARG, "%s", err.c_str());
  for (int i = 0; i < 3; ++i)
    if (xparts) xparts[i] = i < desc->d_x ? pt.parts[i] : 1;
  for (int i = 0; i < 6; ++i) {
    if (off) off[i] = pt.off[i];
    if (len) len[i] = pt.len[i];
  }
  return HD_OK;
}

hd_status hd_halo_chunks(const hd_mesh_desc *desc, int *nchunk, long long *chunk_units, long long *plan) {
  if (!desc || !nchunk) return fail(HD_ERR_ARG, "null argument");
  const int d = desc->d_x + desc->d_v;
  if (desc->d_x < 1 || desc->d_x > 3 || desc->d_v < 1 || desc->d_v > 3 || desc->k < 1 || desc->k > 5)
    return fail(HD_ERR_ARG, "invalid d_x, d_v or k");
  hd::Partition pt;
  std::string err;
  if (!hd::make_partition(*desc, pt, err)) return fail(HD_ERR_ARG, "%s", err.c_str());
  double h[6];
  for (int i = 0; i < d; ++i) h[i] = (desc->hi[i] - desc->lo[i]) / (double)desc->cells[i];
  const int n = desc->k + 1;
  const int pencil_ok = desc->a_lin[6 * 0 + 1] == 0.0;
  const hd::CellGeometry geo = hd::cell_geometry(d, n, (int)pt.len[0], (int)pt.len[1], pt.ncells_local, pencil_ok);
  if (geo.CT < 1) return fail(HD_ERR_UNSUPPORTED, "(d=%d, n=%d) is not in the built kernel set", d, n);
  const long long nunits = geo.pencil ? pt.ncells_local / (pt.len[0] * geo.CT) : pt.ncells_local / geo.CT;
  bool follow_last = geo.pencil && pt.len[d - 1] >= 2;
  for (int j = 0; j < d - 1; ++j) follow_last = follow_last && desc->a_lin[6 * (d - 1) + j] == 0.0;
  hd::HaloDim halo[6];
  for (int i = 0; i < d; ++i) hd::make_halo(*desc, pt, h, i, halo[i]);
  ChunkPlan cp;
  build_chunk_plan(*desc, pt, h, geo, nunits, follow_last, halo, cp);
  *nchunk = cp.nchunk;
  for (int c = 0; c <= cp.nchunk; ++c)
    if (chunk_units) chunk_units[c] = cp.chunk_u[c];
  if (plan)
    for (int c = 0; c < cp.nchunk; ++c)
      for (int i = 0; i < 6; ++i) {
        long long *q = plan + ((size_t)c * 6 + i) * 8;
        const hd_mesh::ChunkHalo &ch = cp.chunk[c];
        q[0] = ch.srq[i];
        q[1] = ch.sr[i][1];
        q[2] = ch.slq[i];
        q[3] = ch.sl[i][1];
        q[4] = ch.rl[i][0];
        q[5] = ch.rl[i][1];
        q[6] = ch.rr[i][0];
        q[7] = ch.rr[i][1];
      }
  return HD_OK;
}

hd_status hd_halo_list(const hd_mesh_desc *desc, int dim, int which, long long *ids, long long *count, int *peer) {
  if (!desc || !count) return fail(HD_ERR_ARG, "null argument");
  if (dim < 0 || dim >= desc->d_x + desc->d_v || which < 0 || which > 3)
    return fail(HD_ERR_ARG, "dim or which out of range");
  hd::Partition pt;
  std::string err;
  if (!hd::make_partition(*desc, pt, err)) return fail(HD_ERR_ARG, "%s", err.c_str());
  const int d = desc->d_x + desc->d_v;
  double h[6];
  for (int i = 0; i < d; ++i) h[i] = (desc->hi[i] - desc->lo[i]) / (double)desc->cells[i];
  hd::HaloDim hd;
  hd::make_halo(*desc, pt, h, dim, hd);
  long long gstride[6], s = 1;
  for (int i = 0; i < d; ++i) {
    gstride[i] = s;
    s *= desc->cells[i];
  }
  // global id of a local cell, optionally shifted by one cell along dim (periodic)
  auto gid = [&](long long cell, int shift) {
    long long g = 0;
    for (int i = 0; i < d; ++i) {
      long long c = pt.off[i] + cell % pt.len[i];
      cell /= pt.len[i];
      if (i == dim) c = (c + shift + desc->cells[i]) % desc->cells[i];
      g += c * gstride[i];
    }
    return g;
  };
  std::vector<long long> out;
  if (hd.active) {
    if (which == 0)
      for (int c : hd.send_left) out.push_back(gid(c, -1));
    if (which == 1)
      for (int c : hd.send_right) out.push_back(gid(c, +1));
    if (which >= 2) {
      // receivers in buffer order: slots [0, n_from_left) are low-face cells, then high-face cells
      long long lstride = 1;
      for (int i = 0; i < dim; ++i) lstride *= pt.len[i];
      const long long plane = hd.slot.size();
      std::vector<long long> byslot(plane, -1);
      for (long long j = 0; j < plane; ++j) {
        const long long lo = j % lstride, hi = j / lstride;
        const bool high = hd.slot[j] >= hd.n_from_left;
        const long long cell = lo + ((high ? pt.len[dim] - 1 : 0) + hi * pt.len[dim]) * lstride;
        byslot[hd.slot[j]] = gid(cell, 0);
      }
      const long long b = which == 2 ? 0 : hd.n_from_left;
      const long long e = which == 2 ? hd.n_from_left : plane;
      for (long long q = b; q < e; ++q) out.push_back(byslot[q]);
    }
  }
  if (peer) *peer = !hd.active ? -1 : (which == 0 || which == 2) ? hd.left : hd.right;
  if (ids) {
    if (*count < (long long)out.size()) return fail(HD_ERR_ARG, "ids too small (%lld < %zu)", *count, out.size());
    for (size_t q = 0; q < out.size(); ++q) ids[q] = out[q];
  }
  *count = (long long)out.size();
  return HD_OK;
}

}  // extern "C"

namespace {

// Launch-dependent kernel parameters of one stage (A mode or an RK stage) and its epoch; every kernel
// launch of the stage (one, or one per v-chunk) shares the epoch, so traces published by an earlier
// chunk's launch are recognised by the later ones.
hd_status begin_stage(hd_mesh *m, hd::CellParams &p, const double *U, double *dU, double *out, int mode, double a,
                      double b, cudaStream_t s) {
  hd_status st = next_epoch(m, p, s);
  if (st != HD_OK) return st;
  p.u = U;
  p.du = dU;
  p.out = out;
  p.mode = mode;
  p.rk_a = a;
  p.rk_b = b;
  return HD_OK;
}
hd_status launch_units(hd_mesh *m, hd::CellParams &p, int u0, int u1, cudaStream_t s) {
  p.u_begin = u0;
  p.u_end = u1;
  p.uctr = m->dbg + 32;
  cudaError_t e = cudaMemsetAsync(p.uctr, 0, sizeof(int), s);
  if (e != cudaSuccess) return cuda_fail(e, "unit counter");
  e = hd::launch_cell_kernel(m->d, m->n, p, s, &m->launches, m->grid);
  if (e != cudaSuccess) return cuda_fail(e, "cell kernel");
#ifdef HD_COUNT
  {  // experiment builds: trace-source counts of this launch (ready published, late published, direct)
    int c[4] = {0, 0, 0, 0};
    cudaStreamSynchronize(s);
    cudaMemcpy(c, m->dbg + 25, sizeof(c), cudaMemcpyDeviceToHost);
    cudaMemset(m->dbg + 25, 0, sizeof(c));
    fprintf(stderr, "HDCOUNT grid %d pub_ready %d pub_late %d direct %d\n", m->grid, c[0], c[1], c[2]);
  }
#endif
  return HD_OK;
}

// One stage of a mesh with its own transport: one launch over all units (one rank), or for nranks > 1
// (NCCL) the v-chunk pipeline: on the mesh's comm stream, after U is ready, chunk c's
// outgoing traces are packed and exchanged (one NCCL group per chunk); on s, chunk c's units run as soon as
// chunk c's traces have arrived -- so the exchange of chunk c+1 overlaps the cell kernel of chunk c.
hd_status launch_stage(hd_mesh *m, hd::CellParams &p, const double *U, double *dU, double *out, int mode, double a,
                       double b, cudaStream_t s) {
  if (m->desc.flux == 1) {
    // central flux: F* = (a.n)(u- + u+)/2 is the mean of the two one-sided operators (every face taking
    // its left cell's trace, resp. its right cell's), each evaluated with the signed speed and weight 1/2
    // (set_dtfac). A mode: v = A_left u / 2, then (kModeAdvAcc) v += A_right u / 2. RK stage: dU <- A_s dU +
    // dt/2 M^-1 A_left U (its U' store is provisional), then dU <- dU + dt/2 M^-1 A_right U, U' <- U + B_s dU.
    hd_status st = begin_stage(m, p, U, dU, out, mode, a, b, s);
    if (st != HD_OK) return st;
    p.sched = m->sched;
    p.schedc = m->schedc;
    st = launch_units(m, p, 0, m->nunits / m->slab, s);
    if (st == HD_OK) st = begin_stage(m, p, U, dU, out, mode == hd::kModeAdvection ? hd::kModeAdvAcc : hd::kModeRK,
                                      mode == hd::kModeAdvection ? 0.0 : 1.0, b, s);
    if (st != HD_OK) return st;
    p.sched = m->sched2;
    p.schedc = m->schedc2;
    st = launch_units(m, p, 0, m->nunits / m->slab, s);
    p.sched = m->sched;
    p.schedc = m->schedc;
    return st;
  }
  hd_status st = begin_stage(m, p, U, dU, out, mode, a, b, s);
  if (st != HD_OK) return st;
  if (m->desc.nranks == 1) return launch_units(m, p, 0, m->nunits / m->slab, s);
  cudaError_t e = cudaEventRecord(m->ev_u, s);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(m->comm, m->ev_u, 0);
  if (e != cudaSuccess) return cuda_fail(e, "halo stream order");
  for (int c = 0; c < m->nchunk; ++c) {
    st = halo_pack(m, p, U, c, m->comm);
    if (st == HD_OK) st = halo_exchange_nccl(m, c, m->comm);
    if (st != HD_OK) return st;
    e = cudaEventRecord(m->ev_chunk[c], m->comm);
    if (e != cudaSuccess) return cuda_fail(e, "halo event");
  }
  for (int c = 0; c < m->nchunk; ++c) {
    e = cudaStreamWaitEvent(s, m->ev_chunk[c], 0);
    if (e != cudaSuccess) return cuda_fail(e, "halo event wait");
    st = launch_units(m, p, m->chunk_u[c], m->chunk_u[c + 1], s);
    if (st != HD_OK) return st;
  }
  return HD_OK;
}

// One stage of P in-process ranks (loopback transport), chunk by chunk: pack chunk c of every rank, copy
// it, run chunk c of every rank -- the same chunk plan, buffers and epochs as the NCCL pipeline, serialised.
hd_status launch_stage_group(hd_mesh **ms, int P, std::vector<hd::CellParams> &ps, const double *const *U,
                             double *const *dU, double *const *out, int mode, double a, double b, cudaStream_t s) {
  for (int r = 0; r < P; ++r) {
    hd_status st = begin_stage(ms[r], ps[r], U[r], dU ? dU[r] : nullptr, out[r], mode, a, b, s);
    if (st != HD_OK) return st;
  }
  for (int c = 0; c < ms[0]->nchunk; ++c) {
    for (int r = 0; r < P; ++r) {
      hd_status st = halo_pack(ms[r], ps[r], U[r], c, s);
      if (st != HD_OK) return st;
    }
    hd_status st = halo_exchange_loopback(ms, P, c, s);
    if (st != HD_OK) return st;
    for (int r = 0; r < P; ++r) {
      st = launch_units(ms[r], ps[r], ms[r]->chunk_u[c], ms[r]->chunk_u[c + 1], s);
      if (st != HD_OK) return st;
    }
  }
  return HD_OK;
}

// HD_DEBUG builds: the non-finite check of an RK stage's output and, at the end of an API call, the
// error word (host synchronises; HD_ERR_STATE with the reason). Release builds: no-ops.
hd_status debug_stage_check(hd_mesh *m, const double *out, cudaStream_t s) {
#ifdef HD_DEBUG
  cudaError_t e = hd::launch_finite_check(out, m->owned_dofs, m->dbg, s);
  if (e != cudaSuccess) return cuda_fail(e, "finite check");
#else
  (void)m;
  (void)out;
  (void)s;
#endif
  return HD_OK;
}
hd_status debug_finish(hd_mesh *const *ms, int P, cudaStream_t s) {
#ifdef HD_DEBUG
  cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "debug synchronise");
  for (int r = 0; r < P; ++r) {
    int w = 0;
    e = cudaMemcpy(&w, ms[r]->dbg, sizeof(int), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(e, "debug word");
    if (w) {
      cudaMemset(ms[r]->dbg, 0, sizeof(int));
      return fail(HD_ERR_STATE, "debug check failed on rank %d:%s%s%s", ms[r]->desc.rank,
                  (w & 1) ? " index out of range" : "", (w & 2) ? " stale halo trace (S:481)" : "",
                  (w & 4) ? " non-finite value after an RK stage (S:508)" : "");
    }
  }
#else
  (void)ms;
  (void)P;
  (void)s;
#endif
  return HD_OK;
}

// Vectors are device pointers the kernels read and write with 16-byte vector accesses.
hd_status check_vec(const void *v, const char *what) {
  if (!v) return fail(HD_ERR_ARG, "null %s", what);
  if (reinterpret_cast<uintptr_t>(v) % 16 != 0) return fail(HD_ERR_ARG, "%s is not 16-byte aligned", what);
  return HD_OK;
}

hd_status check_transport(hd_mesh *m) {
  if (m->desc.nranks > 1 && !m->nccl_comm)
    return fail(HD_ERR_STATE, "multi-rank mesh without NCCL communicator: use the hd_*_group calls (loopback)");
  return HD_OK;
}

hd_status check_bufs(hd_mesh *m, double *buf[3], int *sol, int nsteps, double dt) {
  if (!buf || !sol) return fail(HD_ERR_ARG, "null argument");
  if (*sol < 0 || *sol > 2) return fail(HD_ERR_ARG, "*sol must be 0, 1 or 2");
  if (nsteps < 1) return fail(HD_ERR_ARG, "nsteps must be >= 1");
  if (!std::isfinite(dt)) return fail(HD_ERR_ARG, "dt not finite");
  const size_t bytes = (size_t)m->owned_dofs * sizeof(double);
  for (int i = 0; i < 3; ++i) {
    hd_status st = check_vec(buf[i], "buffer");
    if (st != HD_OK) return st;
    for (int j = 0; j < i; ++j)
      if (overlaps(buf[i], buf[j], bytes)) return fail(HD_ERR_ARG, "buffers %d and %d overlap", j, i);
  }
  return HD_OK;
}

}  // namespace

static hd_status fcl_impl(hd_mesh *m, const double *u, double *v, const double *E, void *stream) {
  if (!m) return fail(HD_ERR_ARG, "null argument");
  hd_status st = check_vec(u, "u");
  if (st == HD_OK) st = check_vec(v, "v");
  if (st != HD_OK) return st;
  if (overlaps(u, v, (size_t)m->owned_dofs * sizeof(double))) return fail(HD_ERR_ARG, "u and v overlap");
  if (m->desc.nranks > 1) return fail(HD_ERR_UNSUPPORTED, "the FCL path is built for single-rank meshes only");
  if (!hd::fcl_supported(m->d, m->n)) return fail(HD_ERR_UNSUPPORTED, "(d=%d, n=%d) cell does not fit the FCL kernel", m->d, m->n);
  const long long fn = m->nd / m->n;
  if (!m->fcl_tr) {
    const size_t tb = (size_t)2 * m->d * m->ncells_local * fn * sizeof(double);
    const size_t gb = (size_t)m->d * m->ncells_local * fn * sizeof(double);
    cudaError_t e = cudaMalloc(&m->fcl_tr, tb);
    if (e == cudaSuccess) e = cudaMalloc(&m->fcl_G, gb);
    if (e != cudaSuccess) {
      cudaGetLastError();
      if (m->fcl_tr) cudaFree(m->fcl_tr);
      m->fcl_tr = nullptr;
      m->fcl_G = nullptr;
      return fail(HD_ERR_OOM, "FCL face buffers (%zu + %zu bytes): %s", tb, gb, cudaGetErrorString(e));
    }
  }
  hd::FclParams p{};
  p.u = u;
  p.v = v;
  p.tr = m->fcl_tr;
  p.G = m->fcl_G;
  p.ncells = m->ncells_local;
  for (int i = 0; i < m->d; ++i) {
    p.L[i] = m->desc.cells[i];
    p.L32[i] = (unsigned)m->desc.cells[i];
    p.lo[i] = m->desc.lo[i];
    p.h[i] = m->h[i];
    p.jdet_h[i] = m->jdet / m->h[i];
    p.a_const[i] = m->desc.a_const[i];
    for (int j = 0; j < m->d; ++j) p.a_lin[i][j] = m->desc.a_lin[6 * i + j];
  }
  for (int a = 0; a < m->n; ++a) {
    p.xi[a] = m->tab.xi[a];
    p.w[a] = m->tab.w[a];
    p.l0[a] = m->tab.tau[1][a];  // tau[1] = l_q(0)
    p.l1[a] = m->tab.tau[0][a];  // tau[0] = l_q(1)
    for (int q = 0; q < m->n; ++q) p.Dw[a][q] = m->tab.Dw[a][q];
  }
  p.flux = m->desc.flux;
  p.E = E;
  p.d_x = m->desc.d_x;
  p.ncx = m->cx_total;
  p.nx = 1;
  for (int i = 0; i < m->desc.d_x; ++i) p.nx *= m->n;
  cudaError_t e = hd::launch_fcl(m->d, m->n, p, (cudaStream_t)stream, &m->launches, m->sms);
  if (e != cudaSuccess) return cuda_fail(e, "FCL kernels");
  return HD_OK;
}

extern "C" {

hd_status hd_apply_advection(hd_mesh *m, const double *u, double *v, double t, void *stream) {
  (void)t;
  if (!m) return fail(HD_ERR_ARG, "null argument");
  hd_status st = check_vec(u, "u");
  if (st == HD_OK) st = check_vec(v, "v");
  if (st != HD_OK) return st;
  if (overlaps(u, v, (size_t)m->owned_dofs * sizeof(double))) return fail(HD_ERR_ARG, "u and v overlap");
  st = check_transport(m);
  if (st == HD_OK) st = ensure_tables(m);
  if (st != HD_OK) return st;
  hd::CellParams p;
  fill_cell_params(m, p);
  set_dtfac(m, p, 1.0);
  st = launch_stage(m, p, u, nullptr, v, hd::kModeAdvection, 0.0, 0.0, (cudaStream_t)stream);
  if (st != HD_OK) return st;
  return debug_finish(&m, 1, (cudaStream_t)stream);
}

// Face-centric loop comparison path (hd_fcl.cu).
hd_status hd_apply_advection_fcl(hd_mesh *m, const double *u, double *v, double t, void *stream) {
  (void)t;
  return fcl_impl(m, u, v, nullptr, stream);
}

// GLL nodal basis <-> Gauss-point values (hd_basis.cu; SURVEY §8(f) NEXT-2, P:228-233, P:509-518, P:556-574;
// DESIGN.md §6 "Basis change")
static hd_status basis_impl(hd_mesh *m, const double *u, double *v, int kind, cudaStream_t s) {
  if (kind < 0 || kind > 3) return fail(HD_ERR_ARG, "kind must be 0..3 (hd_basis_kind)");
  if (!hd::basis_kernel_supported(m->d, m->n))
    return fail(HD_ERR_UNSUPPORTED, "(d=%d, n=%d) cell does not fit the basis-change kernel", m->d, m->n);
  const size_t bytes = (size_t)m->owned_dofs * sizeof(double);
  if (u != v && overlaps(u, v, bytes)) return fail(HD_ERR_ARG, "u and v overlap without being equal");
  double S[4][hd::kMaxN * hd::kMaxN];
  hd::build_basis_tables(m->n, S);
  hd::BasisParams p{};
  p.u = u;
  p.v = v;
  p.ncells = m->ncells_local;
  p.d = m->d;
  for (int e = 0; e < m->n * m->n; ++e) p.S[e] = S[kind][e];
  cudaError_t e = hd::launch_basis_kernel(m->n, p, s, &m->launches, m->sms);
  if (e != cudaSuccess) return cuda_fail(e, "basis change");
  return HD_OK;
}

hd_status hd_basis_change(hd_mesh *m, const double *u, double *v, int kind, void *stream) {
  if (!m) return fail(HD_ERR_ARG, "null argument");
  hd_status st = check_vec(u, "u");
  if (st == HD_OK) st = check_vec(v, "v");
  if (st != HD_OK) return st;
  return basis_impl(m, u, v, kind, (cudaStream_t)stream);
}

hd_status hd_apply_advection_gll(hd_mesh *m, const double *u, double *v, double *work, double t, void *stream) {
  if (!m) return fail(HD_ERR_ARG, "null argument");
  hd_status st = check_vec(u, "u");
  if (st == HD_OK) st = check_vec(v, "v");
  if (st == HD_OK) st = check_vec(work, "work");
  if (st != HD_OK) return st;
  const size_t bytes = (size_t)m->owned_dofs * sizeof(double);
  if (overlaps(u, v, bytes) || overlaps(u, work, bytes) || overlaps(v, work, bytes))
    return fail(HD_ERR_ARG, "u, v and work overlap");
  // P:556-567 steps 2-4: interpolate to the Gauss points, the Gauss-point operator, test with the transpose
  st = basis_impl(m, u, work, HD_GLL_TO_GAUSS, (cudaStream_t)stream);
  if (st == HD_OK) st = hd_apply_advection(m, work, v, t, stream);
  if (st == HD_OK) st = basis_impl(m, v, v, HD_GLL_TO_GAUSS_T, (cudaStream_t)stream);
  return st;
}

hd_status hd_rk_step_gll(hd_mesh *m, double *buf[3], int *sol, double t, double dt, int nsteps, void *stream) {
  if (!m) return fail(HD_ERR_ARG, "null argument");
  hd_status st = check_bufs(m, buf, sol, nsteps, dt);
  if (st != HD_OK) return st;
  // T does not depend on time: one basis change in, the Gauss-basis time loop, one basis change out
  st = basis_impl(m, buf[*sol], buf[*sol], HD_GLL_TO_GAUSS, (cudaStream_t)stream);
  if (st == HD_OK) st = hd_rk_step(m, buf, sol, t, dt, nsteps, stream);
  if (st == HD_OK) st = basis_impl(m, buf[*sol], buf[*sol], HD_GAUSS_TO_GLL, (cudaStream_t)stream);
  return st;
}

hd_status hd_basis_tables(int n, double *gll, double *T) {
  if (n < 2 || n > hd::kMaxN) return fail(HD_ERR_ARG, "n must be in 2..%d", hd::kMaxN);
  double S[4][hd::kMaxN * hd::kMaxN];
  hd::build_basis_tables(n, S);
  if (T)
    for (int k = 0; k < 4; ++k)
      for (int e = 0; e < n * n; ++e) T[k * n * n + e] = S[k][e];
  if (gll) {
    // the GLL points are where the Gauss-to-GLL interpolation of the coordinate x lands
    hd::Tables1D t;
    hd::build_tables(n, t);
    for (int j = 0; j < n; ++j) {
      double x = 0.0;
      for (int q = 0; q < n; ++q) x += S[1][j * n + q] * t.xi[q];
      gll[j] = x;
    }
  }
  return HD_OK;
}

// Vlasov-Poisson (hd_fcl.cu, Eq. equ:vp:close; DESIGN.md §6 "Vlasov-Poisson")
static hd_status vp_setup(hd_mesh *m, hd::VpParams &vp) {
  const int dx = m->desc.d_x, dv = m->desc.d_v, n = m->n;
  if (m->desc.nranks > 1) return fail(HD_ERR_UNSUPPORTED, "the Vlasov-Poisson path is built for single-rank meshes only");
  if (dx != dv || dx > 3) return fail(HD_ERR_UNSUPPORTED, "Vlasov-Poisson needs d_x = d_v <= 3");
  vp = hd::VpParams{};
  vp.d_x = dx;
  vp.n = n;
  vp.nx = 1;
  vp.nv = 1;
  for (int i = 0; i < dx; ++i) vp.nx *= n;
  for (int i = 0; i < dv; ++i) vp.nv *= n;
  if (vp.nv > 216) return fail(HD_ERR_UNSUPPORTED, "too many v nodes per cell");
  vp.ND = (int)m->nd;
  vp.ncx = m->cx_total;
  vp.ncv = m->ncells_local / m->cx_total;
  vp.vol_x = 1.0;
  vp.nmodes = 1;
  for (int i = 0; i < dx; ++i) {
    vp.Lx[i] = m->desc.cells[i];
    vp.lo[i] = m->desc.lo[i];
    vp.h[i] = m->h[i];
    vp.Lbox[i] = m->desc.hi[i] - m->desc.lo[i];
    vp.vol_x *= vp.Lbox[i];
    vp.K[i] = (m->desc.cells[i] - 1) / 2;  // modes below the per-cell Nyquist phase (reading C24)
    vp.nmodes *= 2 * vp.K[i] + 1;
  }
  for (int a = 0; a < n; ++a) {
    vp.xi[a] = m->tab.xi[a];
    vp.w[a] = m->tab.w[a];
  }
  for (int jv = 0; jv < vp.nv; ++jv) {
    double w = 1.0;
    int r = jv;
    for (int i = 0; i < dv; ++i) {
      w *= m->tab.w[r % n] * m->h[dx + i];
      r /= n;
    }
    vp.wv[jv] = w;
  }
  if (!m->vp_rho) {
    const size_t nxn = (size_t)vp.ncx * vp.nx;
    cudaError_t e = cudaMalloc(&m->vp_rho, nxn * sizeof(double));
    if (e == cudaSuccess) e = cudaMalloc(&m->vp_rhohat, (size_t)2 * vp.nmodes * sizeof(double));
    if (e == cudaSuccess) e = cudaMalloc(&m->vp_E, (size_t)dx * nxn * sizeof(double));
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(HD_ERR_OOM, "Vlasov-Poisson field buffers: %s", cudaGetErrorString(e));
    }
  }
  return ensure_tables(m);
}

hd_status hd_vp_fields(hd_mesh *m, const double *f, double *rho, double *E, void *stream) {
  if (!m) return fail(HD_ERR_ARG, "null argument");
  hd_status st = check_vec(f, "f");
  if (st != HD_OK) return st;
  hd::VpParams vp;
  st = vp_setup(m, vp);
  if (st != HD_OK) return st;
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = hd::launch_vp_fields(vp, f, m->vp_rho, m->vp_rhohat, m->vp_E, s, &m->launches, m->sms);
  const size_t nxn = (size_t)vp.ncx * vp.nx;
  if (e == cudaSuccess && rho) e = cudaMemcpyAsync(rho, m->vp_rho, nxn * sizeof(double), cudaMemcpyDeviceToDevice, s);
  if (e == cudaSuccess && E) e = cudaMemcpyAsync(E, m->vp_E, vp.d_x * nxn * sizeof(double), cudaMemcpyDeviceToDevice, s);
  if (e != cudaSuccess) return cuda_fail(e, "Vlasov-Poisson fields");
  return HD_OK;
}

hd_status hd_apply_advection_vp(hd_mesh *m, const double *u, const double *E, double *v, void *stream) {
  if (!m || !E) return fail(HD_ERR_ARG, "null argument");
  if (m->desc.d_x != m->desc.d_v) return fail(HD_ERR_UNSUPPORTED, "Vlasov-Poisson needs d_x = d_v");
  return fcl_impl(m, u, v, E, stream);
}

hd_status hd_vp_rk_step(hd_mesh *m, double *buf[3], double t, double dt, int nsteps, void *stream) {
  (void)t;
  if (!m || !buf) return fail(HD_ERR_ARG, "null argument");
  if (nsteps < 1 || !std::isfinite(dt)) return fail(HD_ERR_ARG, "nsteps must be >= 1 and dt finite");
  const size_t bytes = (size_t)m->owned_dofs * sizeof(double);
  for (int i = 0; i < 3; ++i) {
    hd_status st = check_vec(buf[i], "buf");
    if (st != HD_OK) return st;
    for (int j = 0; j < i; ++j)
      if (overlaps(buf[i], buf[j], bytes)) return fail(HD_ERR_ARG, "buffers overlap");
  }
  hd::VpParams vp;
  hd_status st = vp_setup(m, vp);
  if (st != HD_OK) return st;
  cudaStream_t s = (cudaStream_t)stream;
  hd::StreamParams mp;
  mp.u = buf[2];
  mp.ndofs = m->owned_dofs;
  mp.jdet = m->jdet;
  mp.inverse = 1;
  for (int step = 0; step < nsteps; ++step) {
    for (int stage = 0; stage < 5; ++stage) {
      // E(t_s) from the stage's f ("recomputed once per RK stage"), then M^-1 A(f; a = (v, -E))
      cudaError_t e = hd::launch_vp_fields(vp, buf[0], m->vp_rho, m->vp_rhohat, m->vp_E, s, &m->launches, m->sms);
      if (e != cudaSuccess) return cuda_fail(e, "Vlasov-Poisson fields");
      st = fcl_impl(m, buf[0], buf[2], m->vp_E, stream);
      if (st != HD_OK) return st;
      e = hd::launch_mass_kernel(m->d, m->n, mp, s, &m->launches, m->sms);
      if (e == cudaSuccess)
        e = hd::launch_vp_update(buf[0], buf[1], buf[2], m->owned_dofs, kRkA[stage], kRkB[stage], dt, stage == 0, s,
                                 &m->launches, m->sms);
      if (e != cudaSuccess) return cuda_fail(e, "Vlasov-Poisson stage");
    }
  }
  return HD_OK;
}

hd_status hd_rk_step(hd_mesh *m, double *buf[3], int *sol, double t, double dt, int nsteps, void *stream) {
  (void)t;
  if (!m) return fail(HD_ERR_ARG, "null argument");
  hd_status st = check_bufs(m, buf, sol, nsteps, dt);
  if (st == HD_OK) st = check_transport(m);
  if (st == HD_OK) st = ensure_tables(m);
  if (st != HD_OK) return st;
  hd::CellParams p;
  fill_cell_params(m, p);
  set_dtfac(m, p, dt);
  int iu = *sol, idu = (*sol + 1) % 3, iw = (*sol + 2) % 3;
  for (int step = 0; step < nsteps; ++step) {
    for (int s = 0; s < 5; ++s) {
      st = launch_stage(m, p, buf[iu], buf[idu], buf[iw], s == 0 ? hd::kModeRKFirst : hd::kModeRK, kRkA[s], kRkB[s],
                        (cudaStream_t)stream);
      if (st == HD_OK) st = debug_stage_check(m, buf[iw], (cudaStream_t)stream);
      if (st != HD_OK) return st;
      std::swap(iu, iw);
    }
  }
  *sol = iu;
  return debug_finish(&m, 1, (cudaStream_t)stream);
}

hd_status hd_rk_stage(hd_mesh *m, const double *U, double *dU, double *out, int stage, double dt, void *stream) {
  if (!m) return fail(HD_ERR_ARG, "null argument");
  if (stage < 0 || stage > 4) return fail(HD_ERR_ARG, "stage must be 0..4");
  double *bufs[3] = {const_cast<double *>(U), dU, out};
  int sol = 0;
  hd_status st = check_bufs(m, bufs, &sol, 1, dt);
  if (st == HD_OK) st = check_transport(m);
  if (st == HD_OK) st = ensure_tables(m);
  if (st != HD_OK) return st;
  hd::CellParams p;
  fill_cell_params(m, p);
  set_dtfac(m, p, dt);
  st = launch_stage(m, p, U, dU, out, stage == 0 ? hd::kModeRKFirst : hd::kModeRK, kRkA[stage], kRkB[stage],
                    (cudaStream_t)stream);
  if (st == HD_OK) st = debug_stage_check(m, out, (cudaStream_t)stream);
  if (st != HD_OK) return st;
  return debug_finish(&m, 1, (cudaStream_t)stream);
}

hd_status hd_apply_advection_group(hd_mesh **ms, int P, const double **u, double **v, double t, void *stream) {
  (void)t;
  if (!ms || !u || !v || P < 1) return fail(HD_ERR_ARG, "null argument");
  for (int r = 0; r < P; ++r) {
    if (!ms[r] || !u[r] || !v[r]) return fail(HD_ERR_ARG, "null argument (rank %d)", r);
    if (ms[r]->desc.nranks != P || ms[r]->desc.rank != r) return fail(HD_ERR_ARG, "meshes must be ranks 0..P-1 of P");
    hd_status st = ensure_tables(ms[r]);
    if (st != HD_OK) return st;
  }
  cudaStream_t s = (cudaStream_t)stream;
  std::vector<hd::CellParams> ps(P);
  for (int r = 0; r < P; ++r) {
    fill_cell_params(ms[r], ps[r]);
    set_dtfac(ms[r], ps[r], 1.0);
  }
  hd_status st = launch_stage_group(ms, P, ps, u, nullptr, v, hd::kModeAdvection, 0.0, 0.0, s);
  if (st != HD_OK) return st;
  return debug_finish(ms, P, s);
}

hd_status hd_rk_step_group(hd_mesh **ms, int P, double **bufs, int *sol, double t, double dt, int nsteps,
                           void *stream) {
  (void)t;
  if (!ms || !bufs || !sol || P < 1) return fail(HD_ERR_ARG, "null argument");
  for (int r = 0; r < P; ++r) {
    if (!ms[r]) return fail(HD_ERR_ARG, "null mesh (rank %d)", r);
    if (ms[r]->desc.nranks != P || ms[r]->desc.rank != r) return fail(HD_ERR_ARG, "meshes must be ranks 0..P-1 of P");
    hd_status st = check_bufs(ms[r], bufs + 3 * r, sol, nsteps, dt);
    if (st == HD_OK) st = ensure_tables(ms[r]);
    if (st != HD_OK) return st;
  }
  cudaStream_t s = (cudaStream_t)stream;
  std::vector<hd::CellParams> ps(P);
  for (int r = 0; r < P; ++r) {
    fill_cell_params(ms[r], ps[r]);
    set_dtfac(ms[r], ps[r], dt);
  }
  int iu = *sol, idu = (*sol + 1) % 3, iw = (*sol + 2) % 3;
  std::vector<double *> U(P), DU(P), W(P);
  for (int step = 0; step < nsteps; ++step) {
    for (int st5 = 0; st5 < 5; ++st5) {
      for (int r = 0; r < P; ++r) {
        U[r] = bufs[3 * r + iu];
        DU[r] = bufs[3 * r + idu];
        W[r] = bufs[3 * r + iw];
      }
      hd_status st = launch_stage_group(ms, P, ps, U.data(), DU.data(), W.data(),
                                        st5 == 0 ? hd::kModeRKFirst : hd::kModeRK, kRkA[st5], kRkB[st5], s);
      for (int r = 0; r < P && st == HD_OK; ++r) st = debug_stage_check(ms[r], W[r], s);
      if (st != HD_OK) return st;
      std::swap(iu, iw);
    }
  }
  *sol = iu;
  return debug_finish(ms, P, s);
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
  for (int i = 0; i < m->d; ++i) {
    p.off[i] = m->pt.off[i];
    p.len[i] = m->pt.len[i];
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
