"""GLL nodal basis with Gauss-Legendre quadrature: the paper's default discretisation and its basis change
(Cartesian part).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``). Plain numpy, fp64.

Passages followed:
  * shape functions are tensor products of 1D Lagrange polynomials on the n = k+1
    Gauss-Lobatto-Legendre (GLL) points; integrals use the n-point Gauss-Legendre rule, so the unknowns have
    to be interpolated to the quadrature points first ("basis change").
  * P:556-567, the five steps of a cell integral: 1) gather, 2) interpolate to the quadrature points,
    3) the operation at each quadrature point, 4) test, 5) write back; the basis change is a
    sequence of d 1D interpolation sweeps with the matrix T[q][j] = l^GLL_j(xi^Gauss_q); the testing side
    applies the transposed sweeps.
  With u_G = (T x ... x T) u_L the values at the Gauss points, the GLL weak form is A_L = T^T A_G T and the
  GLL mass matrix M_L = T^T M_G T (A_G, M_G: the Gauss-collocation operator of reading C1, oracle O2), so
  M_L^-1 A_L = T^-1 M_G^-1 A_G T.
GLL points: the end points and the roots of P'_{n-1} (numpy.polynomial.legendre), mapped to [0, 1].
Layout (reading C19): in-cell index j = sum_i m_i n^i, dim 0 fastest.
"""
from __future__ import annotations

import numpy as np

from . import capi, dense


def gll_nodes01(n: int) -> np.ndarray:
    """The n >= 2 Gauss-Lobatto-Legendre points on [0, 1]: 0, 1 and the roots of P'_{n-1}."""
    assert n >= 2
    inner = np.polynomial.legendre.Legendre.basis(n - 1).deriv().roots() if n > 2 else np.zeros(0)
    x = np.concatenate([[-1.0], np.sort(np.real(inner)), [1.0]])
    return 0.5 * (x + 1.0)


def basis_change_matrix(n: int) -> np.ndarray:
    """T[q, j] = l^GLL_j(xi^Gauss_q)."""
    xg, _ = np.polynomial.legendre.leggauss(n)
    xg = 0.5 * (xg + 1.0)
    nodes = gll_nodes01(n)
    T = np.ones((n, n))
    for j in range(n):
        for k in range(n):
            if k != j:
                T[:, j] *= (xg - nodes[k]) / (nodes[j] - nodes[k])
    return T


KINDS = ("gll_to_gauss", "gauss_to_gll", "gll_to_gauss_T", "gauss_to_gll_T")


def matrix_of(n: int, kind: str) -> np.ndarray:
    T = basis_change_matrix(n)
    return {"gll_to_gauss": T, "gauss_to_gll": np.linalg.inv(T), "gll_to_gauss_T": T.T,
            "gauss_to_gll_T": np.linalg.inv(T).T}[kind]


def basis_change(spec: dict, u: np.ndarray, kind: str) -> np.ndarray:
    """Apply the 1D matrix of ``kind`` along every dimension of every cell (d sweeps)."""
    d = spec["d_x"] + spec["d_v"]
    n = spec["k"] + 1
    S = matrix_of(n, kind)
    a = np.asarray(u, float).reshape((-1,) + (n,) * d)      # axis 1 = dim d-1 (slowest) ... axis d = dim 0
    for i in range(d):
        ax = d - i
        a = np.moveaxis(np.tensordot(S, a, axes=([1], [ax])), 0, ax)
    return a.reshape(-1)


def apply_advection_gll(spec: dict, u_gll: np.ndarray, merged: bool = False) -> np.ndarray:
    """v = A_L u (weak form in the GLL basis) by the paper's steps: interpolate to the Gauss points, the
    Gauss-point operator (O2, Alg. 2), test with the transposed interpolation. merged: M_L^-1 A_L u."""
    ug = basis_change(spec, u_gll, "gll_to_gauss")
    if merged:
        return basis_change(spec, capi.apply_advection(spec, ug, merged=True), "gauss_to_gll")
    return basis_change(spec, capi.apply_advection(spec, ug), "gll_to_gauss_T")


def apply_advection_gll_dense(spec: dict, u_gll: np.ndarray, merged: bool = False) -> np.ndarray:
    """The same operator straight from the weak form with the GLL Lagrange basis and an
    over-integrated rule (tier O1, no basis change anywhere): the independent pin of the route above."""
    n = spec["k"] + 1
    A, M = dense.assemble(spec, nodes=gll_nodes01(n))
    v = A @ u_gll
    return np.linalg.solve(M, v) if merged else v


def rk_steps_gll(spec: dict, u_gll: np.ndarray, t: float, dt: float, nsteps: int) -> np.ndarray:
    """LSRK(5,4) steps of du_L/dt = M_L^-1 A_L u_L. T is constant in time, so this is the Gauss-basis
    integration between one basis change in and one out."""
    ug = basis_change(spec, u_gll, "gll_to_gauss")
    return basis_change(spec, capi.rk_steps(spec, ug, t, dt, nsteps), "gauss_to_gll")
