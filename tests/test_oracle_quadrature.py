"""Pins for the oracle's 1D building blocks: Gauss-Legendre by
Newton and the Lagrange basis on its nodes. Pinned against closed forms, against
numpy's independent ``leggauss`` and against exactness boundaries."""
import math

import numpy as np
import pytest

from oracle import capi


def test_n1_n2_closed_forms():
    # n=1 midpoint; n=2 nodes 0.5 -+ 1/(2 sqrt 3), weights 1/2
    x, w = capi.gauss_legendre(1)
    assert x[0] == pytest.approx(0.5, abs=4e-16) and w[0] == pytest.approx(1.0, abs=4e-16)
    x, w = capi.gauss_legendre(2)
    r = 1.0 / (2.0 * math.sqrt(3.0))
    assert np.allclose(x, [0.5 - r, 0.5 + r], atol=4e-16, rtol=0)
    assert np.allclose(w, [0.5, 0.5], atol=4e-16, rtol=0)


def test_n3_n4_n5_closed_forms():
    # classical closed forms of the 3-, 4-, 5-point rules on [-1,1], mapped to [0,1]
    def m(xs, ws):
        return 0.5 * (np.array(xs) + 1.0), 0.5 * np.array(ws)

    s = math.sqrt
    cases = {
        3: m([-s(3 / 5), 0, s(3 / 5)], [5 / 9, 8 / 9, 5 / 9]),
        4: m([-s(3 / 7 + 2 / 7 * s(6 / 5)), -s(3 / 7 - 2 / 7 * s(6 / 5)), s(3 / 7 - 2 / 7 * s(6 / 5)),
              s(3 / 7 + 2 / 7 * s(6 / 5))],
             [(18 - s(30)) / 36, (18 + s(30)) / 36, (18 + s(30)) / 36, (18 - s(30)) / 36]),
        5: m([-s(5 + 2 * s(10 / 7)) / 3, -s(5 - 2 * s(10 / 7)) / 3, 0, s(5 - 2 * s(10 / 7)) / 3,
              s(5 + 2 * s(10 / 7)) / 3],
             [(322 - 13 * s(70)) / 900, (322 + 13 * s(70)) / 900, 128 / 225, (322 + 13 * s(70)) / 900,
              (322 - 13 * s(70)) / 900]),
    }
    for n, (xe, we) in cases.items():
        x, w = capi.gauss_legendre(n)
        assert np.max(np.abs(x - xe)) < 2e-16 * 4, n
        assert np.max(np.abs(w - we)) < 2e-16 * 4, n
    # the n=5 middle weight is 64/225
    assert capi.gauss_legendre(5)[1][2] == pytest.approx(64 / 225, abs=1e-16)


@pytest.mark.parametrize("n", range(1, 13))
def test_matches_numpy_leggauss(n):
    x, w = capi.gauss_legendre(n)
    xr, wr = np.polynomial.legendre.leggauss(n)
    assert np.max(np.abs(x - 0.5 * (xr + 1))) < 1e-15
    assert np.max(np.abs(w - 0.5 * wr)) < 1e-15
    assert abs(w.sum() - 1.0) < 1e-15  # weights sum to 1


@pytest.mark.parametrize("n", range(1, 11))
def test_exactness_boundary(n):
    # S:212 / P:507: exact to degree 2n-1, not exact at 2n
    x, w = capi.gauss_legendre(n)
    for p in range(2 * n):
        assert abs(np.sum(w * x**p) - 1.0 / (p + 1)) < 1e-14, (n, p)
    # degree 2n is not exact: the Gauss error term for f = x^(2n) on [0,1] is
    # I - Q = (n!)^4 / ((2n+1) ((2n)!)^2) (f^(2n) = (2n)!), pinned where it exceeds rounding
    err = 1.0 / (2 * n + 1) - np.sum(w * x ** (2 * n))
    exact = math.factorial(n) ** 4 / ((2 * n + 1) * math.factorial(2 * n) ** 2)
    if exact > 1e-12:
        assert abs(err - exact) < 1e-3 * exact, (n, err, exact)
    assert err > 0


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 6])
def test_lagrange_cardinality_and_unity(n):
    x, _ = capi.gauss_legendre(n)
    for i in range(n):
        val, der = capi.lagrange_eval(n, x[i])
        assert np.max(np.abs(val - np.eye(n)[i])) < 1e-14
        assert abs(der.sum()) < 1e-12  # derivative of partition of unity
    for t in [0.0, 0.3, 1.0]:
        val, der = capi.lagrange_eval(n, t)
        assert abs(val.sum() - 1.0) < 1e-13
        assert abs(der.sum()) < 1e-11
        # reproduce t^p exactly for p < n: sum_j l_j(t) x_j^p = t^p
        for p in range(n):
            assert abs(np.sum(val * x**p) - t**p) < 1e-13


def test_lagrange_derivative_against_finite_difference():
    n = 5
    for t in [0.1, 0.5, 0.77]:
        e = 1e-6
        vp, _ = capi.lagrange_eval(n, t + e)
        vm, _ = capi.lagrange_eval(n, t - e)
        _, der = capi.lagrange_eval(n, t)
        assert np.max(np.abs((vp - vm) / (2 * e) - der)) < 1e-7
