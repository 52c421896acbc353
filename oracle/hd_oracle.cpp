// hd_oracle.cpp -- TEST INFRASTRUCTURE ONLY. Plain, slow, obviously-correct CPU
// reference ("oracle", tier O2 of DESIGN.md) for the DG advection hot path of
// hyper.deal (arXiv 2002.08110). Only tests/, __graft_entry__.smoke() and the
// cpu_baseline / --impl reference legs of bench.py may load this library. It
// shares no code, header, table or constant with the CUDA path.
//
// Citations: P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n.
//
// What it computes (all FP64, periodic Cartesian box, nodal Lagrange basis on the
// n = k+1 Gauss-Legendre points of each 1D reference interval [0,1]):
//   weak form       A(u)_i = (grad phi_i, a u)_cell - sum_faces <phi_i, (a.n) u*>_face
//                   (P:215-227 Eq. into:adv:ref, sign convention P:236; reading C4)
//   inverse mass    u_q <- u_q / (w_q |J|)   (C6/C7)
//   merged op       M^-1 A(u)                (Alg. 2 step 4)
//   LSRK(5,4)       Williamson 2N loop, Carpenter-Kennedy coefficients
//                   (P:3141-3145 cites [Kennedy00]; reading C13)
// The cell routine follows Alg. 2 literally in collocation form:
//   step 1 gather, step 2 t_q = J^-1 a |J| w_q u_q then b_m = sum_q grad phi_m(xi_q).t_q,
//   step 3 all 2d faces with BOTH traces u-, u+ and the flux formula of S:390,
//   step 4 b_q / (w_q |J|), step 5 scatter.
// Deliberately unfolded: no rank-1 folding of the own-face term, both sides of
// every face are evaluated, the upwind choice is made by the S:390 formula.
//
// Build: g++ -O2 -fopenmp -shared -fPIC -o liboracle.so hd_oracle.cpp
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

extern "C" {

// Mesh descriptor of the oracle (its own definition; mirrors the meaning of the
// product's hd_mesh_desc but shares no code with it).
typedef struct {
  int d_x, d_v;          // space dims, d = d_x + d_v in 1..6
  int k;                 // polynomial degree, n = k+1 nodes per dim (k >= 0)
  long long cells[6];    // cells per dim, x dims first
  double lo[6], hi[6];   // periodic box per dim
  double a_const[6];     // a_i(z) = a_const[i] + sum_j a_lin[i][j] z_j
  double a_lin[36];      // row-major [i][j]; a_lin[i][i] must be 0
  int flux;              // 0 upwind, 1 central
} or_desc;

}  // extern "C"

namespace {

// ---- 1D Gauss-Legendre rule on [0,1] by Newton on P_n ---------------
void gauss_legendre01(int n, std::vector<double> &x, std::vector<double> &w) {
  x.assign(n, 0.0);
  w.assign(n, 0.0);
  for (int i = 0; i < n; ++i) {
    // Chebyshev-like initial guess for the i-th largest root of P_n on [-1,1]
    double t = std::cos(M_PI * (i + 0.75) / (n + 0.5));
    double dp = 1.0;
    for (int it = 0; it < 100; ++it) {
      // three-term recurrence: (m+1) P_{m+1} = (2m+1) t P_m - m P_{m-1}
      double p0 = 1.0, p1 = t;
      for (int m = 1; m < n; ++m) {
        double p2 = ((2.0 * m + 1.0) * t * p1 - m * p0) / (m + 1.0);
        p0 = p1;
        p1 = p2;
      }
      double pn = (n == 0) ? 1.0 : p1, pnm1 = p0;
      if (n == 1) { pn = t; pnm1 = 1.0; }
      dp = n * (t * pn - pnm1) / (t * t - 1.0);  // P_n'(t)
      double dt = pn / dp;
      t -= dt;
      if (std::fabs(dt) < 1e-16) break;
    }
    // recompute derivative at the converged root for the weight
    double p0 = 1.0, p1 = t;
    for (int m = 1; m < n; ++m) {
      double p2 = ((2.0 * m + 1.0) * t * p1 - m * p0) / (m + 1.0);
      p0 = p1;
      p1 = p2;
    }
    double pn = p1, pnm1 = p0;
    if (n == 1) { pn = t; pnm1 = 1.0; }
    dp = n * (t * pn - pnm1) / (t * t - 1.0);
    double wt = 2.0 / ((1.0 - t * t) * dp * dp);
    // roots come out in descending t; store ascending on [0,1]
    x[n - 1 - i] = 0.5 * (1.0 + t);
    w[n - 1 - i] = 0.5 * wt;
  }
}

// ---- Lagrange basis on the nodes x (P:400-406 tensor-product nodal basis) -------
double lagrange(const std::vector<double> &x, int j, double t) {
  double v = 1.0;
  for (size_t k = 0; k < x.size(); ++k)
    if ((int)k != j) v *= (t - x[k]) / (x[j] - x[k]);
  return v;
}
double lagrange_deriv(const std::vector<double> &x, int j, double t) {
  double s = 0.0;
  for (size_t l = 0; l < x.size(); ++l) {
    if ((int)l == j) continue;
    double p = 1.0 / (x[j] - x[l]);
    for (size_t k = 0; k < x.size(); ++k)
      if ((int)k != j && k != l) p *= (t - x[k]) / (x[j] - x[k]);
    s += p;
  }
  return s;
}

struct Mesh {
  int d, n;
  long long nd;          // n^d
  long long cells[6];
  long long ncells;
  double h[6], lo[6];
  double a_const[6], a_lin[6][6];
  int flux;
  std::vector<double> xi, w;          // 1D nodes and weights on [0,1]
  std::vector<double> dphi;           // dphi[m*n+q] = l_m'(xi_q)
  std::vector<double> phi0, phi1;     // l_m(0), l_m(1)
  long long pw[7];                    // n^i
};

int setup(const or_desc *ds, Mesh &M) {
  int d = ds->d_x + ds->d_v;
  if (ds->d_x < 0 || ds->d_v < 0 || d < 1 || d > 6 || ds->k < 0 || ds->k > 12) return -1;
  M.d = d;
  M.n = ds->k + 1;
  M.pw[0] = 1;
  for (int i = 1; i <= 6; ++i) M.pw[i] = M.pw[i - 1] * M.n;
  M.nd = M.pw[d];
  M.ncells = 1;
  for (int i = 0; i < d; ++i) {
    if (ds->cells[i] < 1 || !(ds->hi[i] > ds->lo[i])) return -1;
    M.cells[i] = ds->cells[i];
    M.ncells *= ds->cells[i];
    M.lo[i] = ds->lo[i];
    M.h[i] = (ds->hi[i] - ds->lo[i]) / (double)ds->cells[i];
    M.a_const[i] = ds->a_const[i];
    for (int j = 0; j < d; ++j) M.a_lin[i][j] = ds->a_lin[i * 6 + j];
    if (ds->a_lin[i * 6 + i] != 0.0) return -1;  // divergence-free field only
  }
  M.flux = ds->flux;
  gauss_legendre01(M.n, M.xi, M.w);
  int n = M.n;
  M.dphi.assign(n * n, 0.0);
  M.phi0.assign(n, 0.0);
  M.phi1.assign(n, 0.0);
  for (int m = 0; m < n; ++m) {
    M.phi0[m] = lagrange(M.xi, m, 0.0);
    M.phi1[m] = lagrange(M.xi, m, 1.0);
    for (int q = 0; q < n; ++q) M.dphi[m * n + q] = lagrange_deriv(M.xi, m, M.xi[q]);
  }
  return 0;
}

// physical coordinate of 1D node m of cell c in dim i
inline double coord(const Mesh &M, int i, long long c, double xi) { return M.lo[i] + ((double)c + xi) * M.h[i]; }

inline double speed(const Mesh &M, int i, const double *z) {
  double a = M.a_const[i];
  for (int j = 0; j < M.d; ++j) a += M.a_lin[i][j] * z[j];
  return a;
}

// numerical flux: central a.n (u-+u+)/2; upwind adds |a.n| (u- - u+)/2
inline double numflux(double um, double up, double an, int kind) {
  double c = an * 0.5 * (um + up);
  if (kind == 1) return c;
  return c + std::fabs(an) * 0.5 * (um - up);
}

void decompose(const Mesh &M, long long g, long long *c) {
  for (int i = 0; i < M.d; ++i) {
    c[i] = g % M.cells[i];
    g /= M.cells[i];
  }
}
long long compose(const Mesh &M, const long long *c) {
  long long g = 0;
  for (int i = M.d - 1; i >= 0; --i) g = g * M.cells[i] + c[i];
  return g;
}

// Alg. 2 for one cell. nb[2*i+0] = neighbour across face x_i = 0 (left),
// nb[2*i+1] = across x_i = 1 (right). Output b = A(u) on this cell (weak form),
// or M^-1 A(u) if merged.
void cell_apply(const Mesh &M, const long long *cc, const double *u, const double *const *nb, double *out,
                bool merged) {
  const int d = M.d, n = M.n;
  const long long nd = M.nd;
  double Jdet = 1.0;
  for (int i = 0; i < d; ++i) Jdet *= M.h[i];
  std::vector<double> b(nd, 0.0), t(nd * d);
  std::vector<int> mi(d);
  double z[6];
  // step 2: quadrature-point operation t_q = J^-1 a(z_q) |J| w_q u_q (collocation: u_h(xi_q) = u_q)
  for (long long q = 0; q < nd; ++q) {
    long long r = q;
    double wq = 1.0;
    for (int i = 0; i < d; ++i) {
      mi[i] = (int)(r % n);
      r /= n;
      z[i] = coord(M, i, cc[i], M.xi[mi[i]]);
      wq *= M.w[mi[i]];
    }
    for (int i = 0; i < d; ++i) t[q * d + i] = (1.0 / M.h[i]) * speed(M, i, z) * Jdet * wq * u[q];
  }
  // test with the reference gradient: b_m = sum_q grad phi_m(xi_q) . t_q ; with collocation
  // d/dxi_i phi_m(xi_q) = l'_{m_i}(xi_{q_i}) prod_{j!=i} delta_{m_j q_j}
  for (long long m = 0; m < nd; ++m) {
    long long r = m;
    for (int i = 0; i < d; ++i) { mi[i] = (int)(r % n); r /= n; }
    double s = 0.0;
    for (int i = 0; i < d; ++i) {
      long long base = m - (long long)mi[i] * M.pw[i];
      for (int qi = 0; qi < n; ++qi) s += M.dphi[mi[i] * n + qi] * t[(base + qi * M.pw[i]) * d + i];
    }
    b[m] = s;
  }
  // step 3: all 2d faces, both traces, numerical flux, face quadrature
  for (int i = 0; i < d; ++i) {
    double Jface = Jdet / M.h[i];
    for (int side = 0; side < 2; ++side) {
      const double *un = nb[2 * i + side];
      const std::vector<double> &lm = side ? M.phi1 : M.phi0;   // own trace at xi_i = side
      const std::vector<double> &lp = side ? M.phi0 : M.phi1;   // neighbour's trace at the shared face
      double nrm = side ? 1.0 : -1.0;
      // loop over face points: all multi-indices with m_i = 0
      for (long long m = 0; m < nd; ++m) {
        long long r = m;
        for (int j = 0; j < d; ++j) { mi[j] = (int)(r % n); r /= n; }
        if (mi[i] != 0) continue;
        double wf = 1.0;
        for (int j = 0; j < d; ++j) {
          if (j == i) { z[j] = M.lo[j] + ((double)cc[j] + side) * M.h[j]; continue; }
          z[j] = coord(M, j, cc[j], M.xi[mi[j]]);
          wf *= M.w[mi[j]];
        }
        double um = 0.0, up = 0.0;
        for (int j = 0; j < n; ++j) {
          um += lm[j] * u[m + j * M.pw[i]];
          up += lp[j] * un[m + j * M.pw[i]];
        }
        double an = nrm * speed(M, i, z);
        double f = numflux(um, up, an, M.flux);
        for (int j = 0; j < n; ++j) b[m + j * M.pw[i]] -= lm[j] * wf * Jface * f;
      }
    }
  }
  // step 4 (merged operator only): inverse of the diagonal collocated mass w_q |J|
  for (long long m = 0; m < nd; ++m) {
    double val = b[m];
    if (merged) {
      long long r = m;
      double wq = 1.0;
      for (int i = 0; i < d; ++i) { wq *= M.w[r % n]; r /= n; }
      val = val / (wq * Jdet);
    }
    out[m] = val;  // step 5: scatter
  }
}

void apply_all(const Mesh &M, const double *u, double *v, bool merged) {
  const int d = M.d;
#pragma omp parallel for schedule(dynamic, 4)
  for (long long g = 0; g < M.ncells; ++g) {
    long long c[6], cn[6];
    decompose(M, g, c);
    const double *nb[12];
    for (int i = 0; i < d; ++i) {
      for (int s = 0; s < 2; ++s) {
        for (int j = 0; j < d; ++j) cn[j] = c[j];
        cn[i] = (c[i] + (s ? 1 : M.cells[i] - 1)) % M.cells[i];  // periodic (C9)
        nb[2 * i + s] = u + compose(M, cn) * M.nd;
      }
    }
    cell_apply(M, c, u + g * M.nd, nb, v + g * M.nd, merged);
  }
}

void mass_scale(const Mesh &M, double *u, bool inverse) {
  double Jdet = 1.0;
  for (int i = 0; i < M.d; ++i) Jdet *= M.h[i];
#pragma omp parallel for schedule(static)
  for (long long g = 0; g < M.ncells; ++g) {
    for (long long m = 0; m < M.nd; ++m) {
      long long r = m;
      double wq = 1.0;
      for (int i = 0; i < M.d; ++i) { wq *= M.w[r % M.n]; r /= M.n; }
      double mq = wq * Jdet;
      double &x = u[g * M.nd + m];
      x = inverse ? x / mq : x * mq;
    }
  }
}

}  // namespace

extern "C" {

// Carpenter-Kennedy five-stage fourth-order 2N-storage coefficients (reading C13;
// verified by tests/test_oracle_lsrk.py against the order conditions).
static const double RK_A[5] = {0.0, -567301805773.0 / 1357537059087.0, -2404267990393.0 / 2016746695238.0,
                               -3550918686646.0 / 2091501179385.0, -1275806237668.0 / 842570457699.0};
static const double RK_B[5] = {1432997174477.0 / 9575080441755.0, 5161836677717.0 / 13612068292357.0,
                               1720146321549.0 / 2090206949498.0, 3134564353537.0 / 4481467310338.0,
                               2277821191437.0 / 14882151754819.0};
static const double RK_C[5] = {0.0, 1432997174477.0 / 9575080441755.0, 2526269341429.0 / 6820363962896.0,
                               2006345519317.0 / 3224310063776.0, 2802321613138.0 / 2924317926251.0};

int or_rk_coefficients(double *a, double *b, double *c) {
  for (int s = 0; s < 5; ++s) { a[s] = RK_A[s]; b[s] = RK_B[s]; c[s] = RK_C[s]; }
  return 0;
}

int or_gauss_legendre(int n, double *x, double *w) {
  if (n < 1 || n > 64) return -1;
  std::vector<double> xv, wv;
  gauss_legendre01(n, xv, wv);
  for (int i = 0; i < n; ++i) { x[i] = xv[i]; w[i] = wv[i]; }
  return 0;
}

// l_j(t) and l_j'(t) on the Gauss nodes for n points; out[j] for j < n.
int or_lagrange_eval(int n, double t, double *val, double *der) {
  std::vector<double> xv, wv;
  gauss_legendre01(n, xv, wv);
  for (int j = 0; j < n; ++j) { val[j] = lagrange(xv, j, t); der[j] = lagrange_deriv(xv, j, t); }
  return 0;
}

long long or_dof_count(const or_desc *ds) {
  Mesh M;
  if (setup(ds, M)) return -1;
  return M.ncells * M.nd;
}

// v <- A(u) (weak form) if merged == 0, v <- M^-1 A(u) if merged != 0. Global order C19.
int or_apply_advection(const or_desc *ds, const double *u, double *v, int merged) {
  Mesh M;
  if (setup(ds, M)) return -1;
  if (u == v) return -1;
  apply_all(M, u, v, merged != 0);
  return 0;
}

// Per-cell evaluation for sampled parity at sizes where a full vector does not fit
// host memory. cell_ids[c]: global cell id; u_cells: [ncells][2d+1][n^d] holding the
// cell then its neighbours (dim 0 left, dim 0 right, dim 1 left, ...).
int or_apply_advection_cells(const or_desc *ds, long long ncells, const long long *cell_ids, const double *u_cells,
                             double *out, int merged) {
  Mesh M;
  if (setup(ds, M)) return -1;
  const int d = M.d;
#pragma omp parallel for schedule(dynamic, 1)
  for (long long s = 0; s < ncells; ++s) {
    long long c[6];
    decompose(M, cell_ids[s], c);
    const double *base = u_cells + s * (2 * d + 1) * M.nd;
    const double *nb[12];
    for (int f = 0; f < 2 * d; ++f) nb[f] = base + (1 + f) * M.nd;
    cell_apply(M, c, base, nb, out + s * M.nd, merged != 0);
  }
  return 0;
}

int or_apply_inv_mass(const or_desc *ds, double *u) {
  Mesh M;
  if (setup(ds, M)) return -1;
  mass_scale(M, u, true);
  return 0;
}

int or_apply_mass(const or_desc *ds, double *u) {
  Mesh M;
  if (setup(ds, M)) return -1;
  mass_scale(M, u, false);
  return 0;
}

// nsteps LSRK(5,4) steps in the Williamson 2N form:
//   dU <- A_s dU + dt M^-1 A(U, t + c_s dt);  U <- U + B_s dU.
// u: solution (in/out), du, r: caller scratch of the same length.
int or_rk_steps(const or_desc *ds, double *u, double *du, double *r, double t, double dt, int nsteps) {
  Mesh M;
  if (setup(ds, M)) return -1;
  long long N = M.ncells * M.nd;
  for (int step = 0; step < nsteps; ++step) {
    for (int s = 0; s < 5; ++s) {
      apply_all(M, u, r, true);  // the field a does not depend on t in this path
#pragma omp parallel for schedule(static)
      for (long long i = 0; i < N; ++i) {
        du[i] = RK_A[s] * (s == 0 ? 0.0 : du[i]) + dt * r[i];
        u[i] = u[i] + RK_B[s] * du[i];
      }
    }
    t += dt;
  }
  (void)t;
  return 0;
}

int or_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

double or_numerical_flux(double um, double up, double an, int kind) { return numflux(um, up, an, kind); }

}  // extern "C"
