"""Pins of the GLL basis-change oracle (oracle/gll.py):
closed-form GLL points, interpolation exactness, the hand-derived 1D k = 1 operator in the GLL basis
(tests/golden/adv1d_k1_gll_two_cells.txt), the k = 1 GLL mass matrix, and the basis-change route against the
weak form assembled directly in the GLL basis (tier O1, over-integrated, no basis change)."""
import numpy as np
import pytest

from conftest import load_golden
from oracle import capi, dense, gll, lsrk


def spec_of(d_x, d_v, k, cells, lo, hi, a_const, a_lin=None, flux="upwind"):
    d = d_x + d_v
    if a_lin is None:
        a_lin = [[0.0] * d for _ in range(d)]
    return dict(d_x=d_x, d_v=d_v, k=k, cells=cells, lo=lo, hi=hi, a_const=a_const, a_lin=a_lin, flux=flux)


def test_gll_points_closed_forms():
    s5, s37 = np.sqrt(1 / 5), np.sqrt(3 / 7)
    exp = {2: [0, 1], 3: [0, 0.5, 1], 4: [0, (1 - s5) / 2, (1 + s5) / 2, 1],
           5: [0, (1 - s37) / 2, 0.5, (1 + s37) / 2, 1]}
    for n, e in exp.items():
        assert np.max(np.abs(gll.gll_nodes01(n) - np.array(e))) < 1e-15
    x6 = 2 * gll.gll_nodes01(6) - 1     # n = 6: roots of P_5' : 21 x^4 - 14 x^2 + 1 = 0
    inner = x6[1:-1]
    assert np.max(np.abs(21 * inner ** 4 - 14 * inner ** 2 + 1)) < 1e-13


@pytest.mark.parametrize("n", [2, 3, 4, 5, 6])
def test_basis_change_interpolates_polynomials_exactly(n):
    T = gll.basis_change_matrix(n)
    assert np.max(np.abs(T.sum(axis=1) - 1)) < 1e-14            # partition of unity
    xg = 0.5 * (np.polynomial.legendre.leggauss(n)[0] + 1)
    xl = gll.gll_nodes01(n)
    for p in range(n):                                         # degree <= k reproduced, degree n is not
        assert np.max(np.abs(T @ xl ** p - xg ** p)) < 1e-14
    assert np.max(np.abs(T @ xl ** n - xg ** n)) > 1e-4
    for kind, inv in (("gll_to_gauss", "gauss_to_gll"), ("gll_to_gauss_T", "gauss_to_gll_T")):
        assert np.max(np.abs(gll.matrix_of(n, kind) @ gll.matrix_of(n, inv) - np.eye(n))) < 1e-12


def test_basis_change_sweeps_are_the_tensor_product():
    """d sweeps = the Kronecker product matrix applied per cell; a separable polynomial maps to its values
    at the Gauss points (dimension order: dim 0 fastest)."""
    spec = spec_of(2, 1, 2, [2, 1, 2], [0, 0, 0], [1, 1, 1], [1, 1, 1])
    n = 3
    xl, xg = gll.gll_nodes01(n), 0.5 * (np.polynomial.legendre.leggauss(n)[0] + 1)
    f = lambda x, y, z: (1 + x - 2 * x * x) * (0.5 + y * y) * (2 - z)   # noqa: E731
    cell_l = np.array([f(xl[j % 3], xl[(j // 3) % 3], xl[j // 9]) for j in range(27)])
    cell_g = np.array([f(xg[j % 3], xg[(j // 3) % 3], xg[j // 9]) for j in range(27)])
    u = np.tile(cell_l, 4)
    assert np.max(np.abs(gll.basis_change(spec, u, "gll_to_gauss") - np.tile(cell_g, 4))) < 1e-14
    rng = np.random.default_rng(3)
    u = rng.uniform(-1, 1, 4 * 27)
    K = dense._kron_list([gll.matrix_of(n, "gauss_to_gll_T")] * 3)
    assert np.max(np.abs(gll.basis_change(spec, u, "gauss_to_gll_T") - (u.reshape(4, 27) @ K.T).reshape(-1))) < 1e-13


def test_worked_example_gll_closed_form():
    rows = load_golden("adv1d_k1_gll_two_cells.txt")
    expected = np.zeros((4, 4))
    for r, c, v in rows:
        expected[int(r), int(c)] = float(v)
    spec = spec_of(1, 0, 1, [2], [0.0], [1.0], [1.0])
    for fn in (gll.apply_advection_gll, gll.apply_advection_gll_dense):
        got = np.column_stack([fn(spec, np.eye(4)[j], merged=True) for j in range(4)])
        assert np.max(np.abs(got - expected)) < 1e-13, fn.__name__


def test_gll_mass_matrix_k1_closed_form():
    """M_L = T^T M_G T = h [[1/3, 1/6], [1/6, 1/3]] for linear hat functions."""
    spec = spec_of(1, 0, 1, [1], [0.0], [0.7], [1.0])
    M = np.column_stack([gll.basis_change(spec, capi.apply_mass(spec, gll.basis_change(spec, e, "gll_to_gauss")),
                                          "gll_to_gauss_T") for e in np.eye(2)])
    assert np.max(np.abs(M - 0.7 * np.array([[1 / 3, 1 / 6], [1 / 6, 1 / 3]]))) < 1e-15


@pytest.mark.parametrize("d_x,d_v,k,flux", [(1, 1, 1, "upwind"), (1, 1, 2, "upwind"), (1, 1, 3, "central"),
                                            (2, 1, 2, "upwind"), (2, 2, 1, "upwind"), (1, 2, 3, "upwind")])
def test_basis_change_route_equals_direct_gll_weak_form(d_x, d_v, k, flux):
    d = d_x + d_v
    cells = [3, 2, 2, 2][:d]
    a_lin = [[0.0] * d for _ in range(d)]
    a_lin[0][d_x] = 1.0              # a_0 = v_0 (+ const), a_{d_x} depends on x_0: a Vlasov-like field
    a_lin[d_x][0] = -0.5             # sign(a.n) constant per face (reading C11): the n-point face rule is exact
    a_const = [0.3, -0.4, 0.6, 0.8][:d]
    a_const[d_x] = -0.1
    spec = spec_of(d_x, d_v, k, cells, [0.0] * d_x + [0.2] * d_v, [1.0] * d_x + [1.5] * d_v, a_const, a_lin, flux=flux)
    N = capi.dof_count(spec)
    u = np.random.default_rng(10 * d + k).uniform(-1, 1, N)
    for merged in (False, True):
        a = gll.apply_advection_gll(spec, u, merged)
        b = gll.apply_advection_gll_dense(spec, u, merged)
        assert np.max(np.abs(a - b)) <= 1e-12 * np.max(np.abs(b)), merged
    assert np.max(np.abs(gll.apply_advection_gll(spec, np.ones(N)))) < 1e-12       # constant state
    assert abs(gll.apply_advection_gll(spec, u).sum()) < 1e-12 * N                 # conservation


def test_rk_gll_equals_stepping_the_gll_operator():
    """T is constant in time: integrating in the Gauss basis between two basis changes = the 2N scheme on
    M_L^-1 A_L itself (dense GLL operator, tier O1)."""
    spec = spec_of(1, 1, 2, [3, 2], [0.0, -1.0], [1.0, 1.0], [0.0, 0.1], [[0, 1.0], [0.3, 0]])
    N = capi.dof_count(spec)
    u = np.random.default_rng(4).uniform(-1, 1, N)
    A, M = dense.assemble(spec, nodes=gll.gll_nodes01(3))
    L = np.linalg.solve(M, A)
    ref = u
    for s in range(3):
        ref = lsrk.step(lambda w, t: L @ w, ref, 0.01 * s, 0.01)
    got = gll.rk_steps_gll(spec, u, 0.0, 0.01, 3)
    assert np.max(np.abs(got - ref)) < 1e-13
