// hd_tables.cpp -- 1D reference-interval tables of the product path, computed in long double.
//
// Gauss-Legendre nodes/weights on [0,1] ("Gauss--Legendre family ... exact for
// polynomials of degree 2n_q-1"; reading C1/C2: nodal basis on the Gauss points, n_q = n).
// Merged 1D upwind operator for unit speed (P:215-255 with the own-face term folded into the cell
// matrix, SURVEY 8(a) "Operator definition"):
//   a > 0:  (L u)_m = sum_q [w_q l'_m(xi_q) - l_m(1) l_q(1)] / w_m u_q + l_m(0)/w_m * u_left(1)
//   a < 0:  (L u)_m = sum_q [w_q l'_m(xi_q) + l_m(0) l_q(0)] / w_m u_q - l_m(1)/w_m * u_right(0)
// and the d-dimensional merged operator is sum_i (a_i / h_i) L applied along dim i.
#include <cmath>

#include "hd_internal.h"

namespace hd {

namespace {

typedef long double R;

// roots of P_n on (-1,1) by Newton from the asymptotic guess, refined in long double
void legendre_roots(int n, R *x, R *w) {
  const R pi = 3.141592653589793238462643383279502884L;
  for (int i = 0; i < n; ++i) {
    R t = cosl(pi * (4 * i + 3) / (4 * n + 2));
    R pn = 0, dpn = 1;
    for (int it = 0; it < 200; ++it) {
      R pm1 = 1, p = t;  // P_0, P_1
      if (n == 1) { pn = t; pm1 = 1; }
      for (int k = 2; k <= n; ++k) {
        R pk = ((2 * k - 1) * t * p - (k - 1) * pm1) / k;
        pm1 = p;
        p = pk;
      }
      pn = (n == 1) ? t : p;
      R pprev = (n == 1) ? 1 : pm1;
      dpn = n * (pprev - t * pn) / (1 - t * t);
      R step = pn / dpn;
      t -= step;
      if (fabsl(step) < 1e-30L) break;
    }
    // weight 2 / ((1 - t^2) P_n'(t)^2) with P_n' re-evaluated at the root
    R pm1 = 1, p = t;
    for (int k = 2; k <= n; ++k) {
      R pk = ((2 * k - 1) * t * p - (k - 1) * pm1) / k;
      pm1 = p;
      p = pk;
    }
    R pprev = (n == 1) ? 1 : pm1;
    R pv = (n == 1) ? t : p;
    dpn = n * (pprev - t * pv) / (1 - t * t);
    x[i] = t;
    w[i] = 2 / ((1 - t * t) * dpn * dpn);
  }
}

R lag(const R *x, int n, int j, R t) {
  R v = 1;
  for (int k = 0; k < n; ++k)
    if (k != j) v *= (t - x[k]) / (x[j] - x[k]);
  return v;
}

R lag_d(const R *x, int n, int j, R t) {
  R s = 0;
  for (int l = 0; l < n; ++l) {
    if (l == j) continue;
    R p = 1 / (x[j] - x[l]);
    for (int k = 0; k < n; ++k)
      if (k != j && k != l) p *= (t - x[k]) / (x[j] - x[k]);
    s += p;
  }
  return s;
}

}  // namespace

void build_tables(int n, Tables1D &t) {
  R xr[kMaxN], wr[kMaxN], x01[kMaxN], w01[kMaxN];
  legendre_roots(n, xr, wr);
  // roots come out descending in [-1,1]; map ascending onto [0,1]
  for (int i = 0; i < n; ++i) {
    x01[n - 1 - i] = (1 + xr[i]) / 2;
    w01[n - 1 - i] = wr[i] / 2;
  }
  for (int i = 0; i < kMaxN; ++i) {
    t.xi[i] = i < n ? (double)x01[i] : 0.0;
    t.w[i] = i < n ? (double)w01[i] : 0.0;
  }
  R l0[kMaxN], l1[kMaxN];
  for (int m = 0; m < n; ++m) {
    l0[m] = lag(x01, n, m, 0);
    l1[m] = lag(x01, n, m, 1);
  }
  for (int s = 0; s < 2; ++s)
    for (int m = 0; m < kMaxN; ++m) {
      t.lam[s][m] = 0;
      t.tau[s][m] = 0;
      for (int q = 0; q < kMaxN; ++q) t.K[s][m][q] = 0;
      for (int q = 0; q < kMaxN && s == 0; ++q) t.Dw[m][q] = 0;
    }
  for (int m = 0; m < n; ++m) {
    for (int q = 0; q < n; ++q) {
      R vol = w01[q] * lag_d(x01, n, m, x01[q]);
      t.Dw[m][q] = (double)vol;
      t.K[0][m][q] = (double)((vol - l1[m] * l1[q]) / w01[m]);
      t.K[1][m][q] = (double)((vol + l0[m] * l0[q]) / w01[m]);
    }
    t.lam[0][m] = (double)(l0[m] / w01[m]);
    t.lam[1][m] = (double)(-l1[m] / w01[m]);
    t.tau[0][m] = (double)l1[m];
    t.tau[1][m] = (double)l0[m];
  }
}

// Basis change between the GLL nodal basis (the paper's default shape functions) and the values at
// the n Gauss points. GLL points: -1, 1 and the roots of P'_{n-1}, by Newton on
// q(x) = P'_{n-1}(x) with q' from the Legendre equation (1 - x^2) P'' = 2 x P' - m (m + 1) P.
// S[0] = T, T[q][j] = l^GLL_j(xi^Gauss_q); S[1] = T^-1 = l^Gauss_q(x^GLL_j) (both bases span P_k, so the inverse
// is the interpolation the other way round, no linear solve); S[2] = T^T; S[3] = T^-T. Row-major [out][in].
void build_basis_tables(int n, double S[4][kMaxN * kMaxN]) {
  const R pi = 3.141592653589793238462643383279502884L;
  R xr[kMaxN], wr[kMaxN], xg[kMaxN], xl[kMaxN];
  legendre_roots(n, xr, wr);
  for (int i = 0; i < n; ++i) xg[n - 1 - i] = (1 + xr[i]) / 2;
  const int m = n - 1;
  xl[0] = 0;
  xl[n - 1] = 1;
  for (int i = 1; i < n - 1; ++i) {
    R t = -cosl(pi * i / m);  // Chebyshev-Lobatto guess, ascending
    for (int it = 0; it < 200; ++it) {
      R pm1 = 1, p = t;
      for (int k = 2; k <= m; ++k) {
        R pk = ((2 * k - 1) * t * p - (k - 1) * pm1) / k;
        pm1 = p;
        p = pk;
      }
      const R dp = m * (pm1 - t * p) / (1 - t * t);                    // P'_m
      const R ddp = (2 * t * dp - (R)m * (m + 1) * p) / (1 - t * t);   // P''_m
      const R step = dp / ddp;
      t -= step;
      if (fabsl(step) < 1e-30L) break;
    }
    xl[i] = (1 + t) / 2;
  }
  for (int k = 0; k < 4; ++k)
    for (int e = 0; e < kMaxN * kMaxN; ++e) S[k][e] = 0;
  for (int q = 0; q < n; ++q)
    for (int j = 0; j < n; ++j) {
      const R t = lag(xl, n, j, xg[q]);   // T[q][j]
      const R ti = lag(xg, n, q, xl[j]);  // T^-1[j][q]
      S[0][q * n + j] = (double)t;
      S[2][j * n + q] = (double)t;
      S[1][j * n + q] = (double)ti;
      S[3][q * n + j] = (double)ti;
    }
}

}  // namespace hd
