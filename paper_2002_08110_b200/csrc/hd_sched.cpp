// hd_sched.cpp -- the static schedule of the fused cell kernel (DESIGN.md §6 "Schedule"), built once per
// mesh on the host. Round 1 decoded units, cells and trace sources on the device for every group (one
// lane per (cell, dim), divergent, ~20 instructions per DoF); the decisions are all static, so they are
// made here and stored as one 32-byte SchedDim record per (group, cell slot, dim).
//
// Central flux (NEXT-3): the schedule can force every dim's "upwind" side (forced = 0: the left neighbour,
// 1: the right one) -- the two one-sided operators whose mean is the central-flux operator;
// the traversal then follows the forced direction.
//
// Work decomposition (unchanged from round 1):
//   * pencil mode (CT | L_1, a_0 independent of z_1): a group is CT cells at one c_0 from CT adjacent
//     dim-0 pencils; a unit is those CT pencils, processed by ONE CTA group by group, upwind -> downwind
//     along dim 0. Units are ordered lexicographically over (t_1, ..., t_{d-1}) with every dim whose
//     speed sign depends only on slower dims ("follows") traversed upwind -> downwind, so the upwind
//     neighbour along such a dim is an earlier unit. A unit starts at step (-skew * sum_j t_j) mod GPU:
//     its upwind neighbours in the same round of units run `skew` groups ahead.
//   * multi-pencil mode (L_0 | CT): a group (= a unit) holds whole pencils.
//   * chunk mode (CT | L_0, a_0 depends on z_1): a group is CT consecutive cells of one pencil.
// Trace sources per (cell, dim) (the upwind neighbour's n^(d-1)-value trace, P:1086-1094 with the
// rank-1 folding of DESIGN.md §6): the dim-0 carry of the previous step (smem), an in-group neighbour
// (smem), a trace published by an earlier unit (checked against its progress flag at run time, else a
// direct read), the halo receive buffer (multi-rank), or a direct read of the neighbour cell.
#include <algorithm>
#include <cmath>
#include <vector>

#include "hd_internal.h"

namespace hd {
namespace {

struct Geo {
  int d, CT, GPU, pencil, skew, slab;
  int forced;  // -1: the sign of a_i decides the upwind side; 0 / 1: every dim takes its left / right neighbour
  long long L[kMaxD], lstride[kMaxD], ustride[kMaxD], off[kMaxD];
  int follow[kMaxD], pub[kMaxD], xsplit[kMaxD];
  long long UC;
  const hd_mesh *m;
  // wavefront unit order (pencil mode, one v-chunk): order[u] = the lexicographic index of unit u, rank =
  // its inverse; empty = lexicographic
  std::vector<long long> order, rank;
};

// a_i at the lower corner of the cell with local coordinates c and its sign on the cell (evaluated at the
// centre; constant on the cell by reading C11). The device pack kernel evaluates the same fma sequence,
// so the values agree bitwise.
void cell_speed(const Geo &g, int i, const long long *c, double &base, int &sg) {
  const hd_mesh_desc &ds = g.m->desc;
  double ab = ds.a_const[i], half = 0.0;
  for (int j = 0; j < g.d; ++j) {
    ab = std::fma(ds.a_lin[6 * i + j], std::fma((double)(c[j] + g.off[j]), g.m->h[j], ds.lo[j]), ab);
    half = std::fma(ds.a_lin[6 * i + j], 0.5 * g.m->h[j], half);
  }
  base = ab;
  sg = g.forced >= 0 ? g.forced : (ab + half) < 0.0 ? 1 : 0;
}

struct Unit {
  long long c[kMaxD];
  long long base;
  int dir0, skew;
  long long pu[kMaxD];
  int pdir0[kMaxD], pskew[kMaxD];
};

// traversal coordinates of pencil-mode unit u -> the unit's first cell coordinates, dim-0 direction, start
long long pencil_decode(const Geo &g, long long u, long long *c, int &dir0, int &skew) {
  long long base = 0, tsum = 0;
  if (!g.order.empty()) u = g.order[(size_t)u];
  for (int j = 0; j < kMaxD; ++j) c[j] = 0;
  for (int j = g.d - 1; j >= 1; --j) {
    const long long ext = j == 1 ? g.L[1] / g.CT : g.L[j];
    const long long tj = (u / g.ustride[j]) % ext;
    tsum += tj;
    int neg = 0;
    if (g.follow[j]) {
      double b;
      cell_speed(g, j, c, b, neg);  // faster coordinates are still 0: a_j does not depend on them
    }
    const long long cj = neg ? ext - 1 - tj : tj;
    c[j] = j == 1 ? cj * g.CT : cj;
    base += c[j] * g.lstride[j];
  }
  double b0;
  cell_speed(g, 0, c, b0, dir0);
  skew = (int)((g.GPU - (g.skew * tsum) % g.GPU) % g.GPU);
  return base;
}

long long unit_of(const Geo &g, const long long *c) {
  long long cc[kMaxD] = {0, 0, 0, 0, 0, 0}, u = 0;
  for (int j = g.d - 1; j >= 1; --j) {
    int neg = 0;
    if (g.follow[j]) {
      double b;
      cell_speed(g, j, cc, b, neg);
    }
    cc[j] = c[j];
    const long long ext = j == 1 ? g.L[1] / g.CT : g.L[j];
    const long long cj = j == 1 ? c[1] / g.CT : c[j];
    u += (neg ? ext - 1 - cj : cj) * g.ustride[j];
  }
  return g.rank.empty() ? u : g.rank[(size_t)u];
}

int step_group(const Geo &g, int gi, int dir0, int skew) {
  const int q = (gi + skew) % g.GPU;
  return dir0 ? g.GPU - 1 - q : q;
}
int group_step(const Geo &g, int grp, int dir0, int skew) {
  const int gg = dir0 ? g.GPU - 1 - grp : grp;
  return (gg - skew + g.GPU) % g.GPU;
}

void decode_unit(const Geo &g, long long u, Unit &ui) {
  ui.base = pencil_decode(g, u, ui.c, ui.dir0, ui.skew);
  for (int j = 0; j < kMaxD; ++j) {
    ui.pu[j] = -1;
    ui.pdir0[j] = 0;
    ui.pskew[j] = 0;
  }
  for (int j = 1; j < g.d; ++j) {
    if (!g.pub[j]) continue;
    // the upwind neighbour along j of every cell of this pencil sits in one pencil (a_j does not depend on
    // z_0 or z_j): its unit, direction and start
    double b;
    int sg;
    cell_speed(g, j, ui.c, b, sg);
    long long cn[kMaxD];
    for (int q = 0; q < kMaxD; ++q) cn[q] = ui.c[q];
    if (j == 1) cn[1] = sg ? ui.c[1] + g.CT - 1 : ui.c[1];  // the unit's upwind end along dim 1
    cn[j] += sg ? 1 : -1;
    if (cn[j] >= 0 && cn[j] < g.L[j]) {
      const long long pu = unit_of(g, cn);
      long long pc[kMaxD];
      int pd, ps;
      pencil_decode(g, pu, pc, pd, ps);
      if (pu < u) {  // an earlier unit: published in time (same round: `skew` steps ahead)
        ui.pu[j] = pu;
        ui.pdir0[j] = pd;
        ui.pskew[j] = ps;
      }
    }
  }
}

}  // namespace

void build_schedule(const hd_mesh &m, std::vector<SchedDim> &out, std::vector<SchedCell> &cells, int forced) {
  Geo g{};
  g.m = &m;
  g.forced = forced;
  g.d = m.d;
  g.CT = m.geo.CT;
  g.GPU = m.geo.GPU;
  g.pencil = m.geo.pencil;
  g.skew = m.skew;
  g.slab = m.slab;
  long long ls = 1, us = 1;
  for (int i = 0; i < g.d; ++i) {
    g.L[i] = m.pt.len[i];
    g.off[i] = m.pt.off[i];
    g.lstride[i] = ls;
    ls *= g.L[i];
    if (i >= 1) {
      g.ustride[i] = us;
      us *= (i == 1 && g.pencil) ? g.L[i] / g.CT : g.L[i];
    }
    g.follow[i] = m.follow[i];
    g.pub[i] = m.pub[i];
    g.xsplit[i] = m.pt.parts[i] > 1 ? 1 : 0;
  }
  g.UC = g.pencil ? g.L[0] * g.CT : g.CT;
  if (g.pencil && m.nchunk == 1 && m.nunits > 1) {
    // Wavefront order: units sorted by the sum of their traversal coordinates (stable). Every upwind
    // neighbour of a unit lies on the previous hyperplane, so it still comes earlier, but units dealt
    // together (one round of CTAs) are rarely neighbours: the producer of a published trace has usually
    // finished its whole pencil, and the skew seams (a same-round consumer's first `skew` steps, whose
    // producer processes those cells last) become rare. Slab super-units (slab > 1): the key leaves out
    // t_1, so the slab's pencils (t_1 = 0 .. slab-1, lexicographic index fastest in t_1) stay consecutive
    // -- kernel unit U = pencil units U*slab .. U*slab + slab-1, run one after the other.
    const long long nu = m.nunits;
    std::vector<int> key((size_t)nu);
    int kmax = 0;
    for (long long u = 0; u < nu; ++u) {
      int t = 0;
      for (int j = g.slab > 1 ? 2 : 1; j < g.d; ++j) {
        const long long ext = (j == 1 && g.pencil) ? g.L[1] / g.CT : g.L[j];
        t += (int)((u / g.ustride[j]) % ext);
      }
      key[(size_t)u] = t;
      kmax = std::max(kmax, t);
    }
    std::vector<long long> start((size_t)kmax + 2, 0);
    for (long long u = 0; u < nu; ++u) ++start[(size_t)key[(size_t)u] + 1];
    for (int k = 0; k <= kmax; ++k) start[(size_t)k + 1] += start[(size_t)k];
    g.order.assign((size_t)nu, 0);
    g.rank.assign((size_t)nu, 0);
    for (long long u = 0; u < nu; ++u) {
      const long long pos = start[(size_t)key[(size_t)u]]++;
      g.order[(size_t)pos] = u;
      g.rank[(size_t)u] = pos;
    }
  }
  const int d = g.d, CT = g.CT, GPU = g.GPU;
  out.assign((size_t)m.nunits * GPU * CT * d, SchedDim{});
  cells.assign((size_t)m.nunits * GPU * CT, SchedCell{});
  Unit ui{};
  for (int j = 0; j < kMaxD; ++j) ui.pu[j] = -1;
  for (long long u = 0; u < m.nunits; ++u) {
    if (g.pencil) decode_unit(g, u, ui);
    for (int gi = 0; gi < GPU; ++gi) {
      for (int k = 0; k < CT; ++k) {
        long long c[kMaxD] = {0, 0, 0, 0, 0, 0};
        long long first;
        if (g.pencil) {
          for (int j = 0; j < kMaxD; ++j) c[j] = ui.c[j];
          const int grp = step_group(g, gi, ui.dir0, ui.skew);
          c[0] = grp;
          c[1] += k;
          first = ui.base + grp;
        } else {
          first = u * CT;
          long long rr = first + k;
          for (int j = 0; j < d; ++j) {
            c[j] = rr % g.L[j];
            rr /= g.L[j];
          }
        }
        long long cell = 0;
        for (int j = 0; j < d; ++j) cell += c[j] * g.lstride[j];
        const long long cu = g.pencil ? k * g.L[0] + c[0] : k;
        SchedCell &sc = cells[((size_t)u * GPU + gi) * CT + k];
        sc.cell = (int)cell;
        sc.oslot = (int)(u * g.UC + cu);
        for (int i = 0; i < d; ++i) {
          SchedDim &r = out[(((size_t)u * GPU + gi) * CT + k) * d + i];
          double base;
          int sg;
          cell_speed(g, i, c, base, sg);
          r.base = base;
          r.sg = (unsigned char)sg;
          const int up = sg ? 1 : -1;
          long long cn = c[i] + up;
          const bool outside = cn < 0 || cn >= g.L[i];
          if (cn < 0) cn += g.L[i];
          if (cn >= g.L[i]) cn -= g.L[i];
          const long long nbcell = cell + (cn - c[i]) * g.lstride[i];
          unsigned char src = kSrcDirect, o = kOutNone;
          long long slot = 0;
          int pflag = -1, need = 0;
          if (i == 0 && g.pencil && gi < GPU - 1) o = kOutCarry;  // feeds the carry of the next step
          if (i > 0 && g.pub[i]) {
            // downwind neighbour inside the local box and outside this group: publish
            const long long cd = c[i] - up;
            const bool in_group = g.pencil && i == 1 && k - up >= 0 && k - up < CT;
            if (cd >= 0 && cd < g.L[i] && !in_group) o = kOutPub;
          }
          if (outside && g.xsplit[i]) {
            // the upwind neighbour lives on another rank: its trace arrives in the halo buffer
            src = kSrcHalo;
            const long long lsi = g.lstride[i];
            slot = m.halo[i].slot[(size_t)((cell % lsi) + (cell / (lsi * g.L[i])) * lsi)];
          } else if (i == 0 && g.pencil) {
            if (gi > 0) src = kSrcCarry;  // the previous step processed the upwind neighbour along dim 0
          } else if (g.pencil && i == 1 && k + up >= 0 && k + up < CT) {
            src = kSrcGroup;  // the neighbour pencil is in this group
            slot = k + up;
          } else if (!g.pencil && nbcell >= first && nbcell < first + CT) {
            src = kSrcGroup;
            slot = nbcell - first;
          } else if (g.pub[i] && !outside && ui.pu[i] >= 0) {
            // published by an earlier unit: the flag value meaning "the step that processed the
            // neighbour's group is done", and the neighbour's slot in the producer unit (same pencil and
            // c_0, except along dim 1 where it is the other end of the neighbouring block)
            src = kSrcPub;
            // flags and steps are per kernel unit: a slab super-unit runs its pencils one after the other
            pflag = (int)(ui.pu[i] / g.slab);
            need = (int)(ui.pu[i] % g.slab) * GPU + group_step(g, (int)c[0], ui.pdir0[i], ui.pskew[i]) + 1;
            const long long kn = (g.pencil && i == 1) ? (k + up + CT) % CT : k;
            slot = ui.pu[i] * g.UC + (g.pencil ? kn * g.L[0] + c[0] : kn);
          }
          r.src = src;
          r.out = o;
          r.nb = (int)nbcell;
          r.slot = (int)slot;
          r.pflag = pflag;
          r.need = need;
        }
      }
    }
  }
}

}  // namespace hd
