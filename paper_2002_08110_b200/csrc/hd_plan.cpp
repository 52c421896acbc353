// hd_plan.cpp -- host-only x-space partition and halo plan.
//
// Partition: the ranks form a grid parts[0] x ... x parts[d-1] over the cells; automatically only x dims are
// split (every v-cell rank-local), an explicit hd_mesh_desc.vparts also splits v dims (the checkerboard x-v
// partition of P:913-948). Automatic: xparts[0] x ... x xparts[d_x-1] over the x-cells (x-slabs when only
// the slowest x dim is split, x-blocks otherwise); every v-cell is rank-local ("phase-space
// partition", with the v part undivided), so v-faces and M^-1 never communicate. Each rank owns the
// box [off, off + len) of the global Cartesian cell grid, stored lexicographically (first axis fastest,
// reading C19) -- with one rank this is exactly the global order.
//
// Halo (a2): with upwind fluxes a cell needs only its UPWIND neighbour's trace (n^(d-1) values, 1/n of a
// cell). Across an x-face between ranks along dim i, the sign of a_i is the same on both sides (a_i does
// not depend on z_i), so for every position j of the face plane exactly one trace crosses: from the left
// rank when a_i > 0, from the right rank when a_i < 0. The receiving buffer of dim i holds the traces
// for the positions with a_i > 0 (from the left, in plane order) followed by those with a_i < 0 (from the
// right, in plane order); both sides enumerate the same positions in the same order, so the message
// layouts agree without exchanging indices.
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "hd_internal.h"

namespace hd {

// sign of a_i on the cell with GLOBAL coordinates cg (1: a_i < 0). The device evaluates the same
// expression (hd_cell.cuh cell_speed) with explicit fma, so the decisions agree bitwise.
int host_cell_sign(const hd_mesh_desc &ds, const double *h, int d, int i, const long long *cg) {
  double ab = ds.a_const[i], half = 0.0;
  for (int j = 0; j < d; ++j) {
    ab = std::fma(ds.a_lin[6 * i + j], std::fma((double)cg[j], h[j], ds.lo[j]), ab);
    half = std::fma(ds.a_lin[6 * i + j], 0.5 * h[j], half);
  }
  return (ab + half) < 0.0 ? 1 : 0;
}

bool make_partition(const hd_mesh_desc &ds, Partition &pt, std::string &err) {
  const int d = ds.d_x + ds.d_v;
  const int P = ds.nranks;
  pt = Partition();
  pt.d = d;
  pt.d_x = ds.d_x;
  pt.P = P;
  pt.rank = ds.rank;
  for (int i = 0; i < 6; ++i) pt.parts[i] = 1;
  bool explicit_parts = false;
  for (int i = 0; i < 3; ++i) explicit_parts |= ds.xparts[i] > 0 || ds.vparts[i] > 0;
  if (explicit_parts) {
    long long prod = 1;
    for (int i = 0; i < d; ++i) {
      const int given = i < ds.d_x ? ds.xparts[i] : ds.vparts[i - ds.d_x];
      const int pi = given > 0 ? given : 1;
      if (ds.cells[i] % pi != 0) {
        err = "the ranks along dim " + std::to_string(i) + " must divide cells[" + std::to_string(i) + "]";
        return false;
      }
      pt.parts[i] = pi;
      prod *= pi;
    }
    if (prod != P) {
      err = "product of xparts and vparts must equal nranks";
      return false;
    }
  } else if (P > 1) {
    // choose xparts (p_i | cells_i, prod = P) minimising the halo volume sum_{i: p_i > 1} |box| / len_i;
    // ties prefer splitting slower dims (x-slabs when possible)
    const int nx = ds.d_x;
    double best = -1.0;
    long long best_key = 0;
    int bp[3] = {1, 1, 1};
    for (int p0 = 1; p0 <= P; ++p0)
      for (int p1 = 1; p1 <= P; ++p1)
        for (int p2 = 1; p2 <= P; ++p2) {
          const int pp[3] = {p0, p1, p2};
          if ((long long)p0 * p1 * p2 != P) continue;
          bool ok = true;
          for (int i = 0; i < 3; ++i) {
            if (i >= nx && pp[i] != 1) ok = false;
            if (i < nx && ds.cells[i] % pp[i]) ok = false;
          }
          if (!ok) continue;
          double box = 1.0;
          for (int i = 0; i < d; ++i) box *= (double)ds.cells[i] / (i < 3 ? pp[i] : 1);
          double halo = 0.0;
          for (int i = 0; i < nx; ++i)
            if (pp[i] > 1) halo += box / ((double)ds.cells[i] / pp[i]);
          const long long key = (long long)p2 * 1000 + p1;  // larger = slower dims split more
          if (best < 0.0 || halo < best * (1 - 1e-12) || (halo <= best * (1 + 1e-12) && key > best_key)) {
            best = halo;
            best_key = key;
            bp[0] = p0;
            bp[1] = p1;
            bp[2] = p2;
          }
        }
    if (best < 0.0) {
      err = "nranks cannot be factored over the x dims (need p_i | cells_i, prod p_i = nranks)";
      return false;
    }
    for (int i = 0; i < 3; ++i) pt.parts[i] = bp[i];
  }
  int r = ds.rank;
  for (int i = 0; i < d; ++i) {
    pt.bcoord[i] = r % pt.parts[i];
    r /= pt.parts[i];
  }
  pt.ncells_local = 1;
  for (int i = 0; i < d; ++i) {
    pt.len[i] = ds.cells[i] / pt.parts[i];
    pt.off[i] = pt.bcoord[i] * pt.len[i];
    pt.ncells_local *= pt.len[i];
  }
  return true;
}

int neighbour_rank(const Partition &pt, int i, int delta) {
  int bc[6];
  for (int j = 0; j < 6; ++j) bc[j] = pt.bcoord[j];
  bc[i] = (bc[i] + delta + pt.parts[i]) % pt.parts[i];
  int r = 0;
  for (int j = pt.d - 1; j >= 0; --j) r = r * pt.parts[j] + bc[j];
  return r;
}

void make_halo(const hd_mesh_desc &ds, const Partition &pt, const double *h, int i, HaloDim &hd) {
  const int d = pt.d;
  hd = HaloDim();
  hd.active = pt.parts[i] > 1;
  if (!hd.active) return;
  hd.left = neighbour_rank(pt, i, -1);
  hd.right = neighbour_rank(pt, i, +1);
  long long lstride[6], s = 1;
  for (int j = 0; j < d; ++j) {
    lstride[j] = s;
    s *= pt.len[j];
  }
  const long long plane = pt.ncells_local / pt.len[i];
  hd.slot.assign(plane, -1);
  std::vector<int> sg(plane);
  // plane positions in lexicographic order of the local box without dim i
  for (long long j = 0; j < plane; ++j) {
    long long rr = j, cg[6];
    for (int k = 0; k < d; ++k) {
      if (k == i) {
        cg[k] = pt.off[k];
        continue;
      }
      cg[k] = pt.off[k] + rr % pt.len[k];
      rr /= pt.len[k];
    }
    sg[j] = host_cell_sign(ds, h, d, i, cg);
  }
  long long n0 = 0, n1 = 0;
  for (long long j = 0; j < plane; ++j) (sg[j] ? n1 : n0) += 1;
  hd.n_from_left = n0;
  hd.n_from_right = n1;
  long long a = 0, b = n0;
  for (long long j = 0; j < plane; ++j) hd.slot[j] = (int)(sg[j] ? b++ : a++);
  // local cell index of plane position j on the low (c_i = 0) or high (c_i = len_i - 1) face
  auto face_cell = [&](long long j, bool high) {
    long long rr = j, cell = 0;
    for (int k = 0; k < d; ++k) {
      if (k == i) {
        cell += (high ? pt.len[k] - 1 : 0) * lstride[k];
        continue;
      }
      cell += (rr % pt.len[k]) * lstride[k];
      rr /= pt.len[k];
    }
    return cell;
  };
  for (long long j = 0; j < plane; ++j) {
    if (sg[j]) hd.send_left.push_back((int)face_cell(j, false));   // a_i < 0: my low face feeds the left rank
    else hd.send_right.push_back((int)face_cell(j, true));         // a_i > 0: my high face feeds the right rank
  }
}

}  // namespace hd
