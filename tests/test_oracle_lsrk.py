"""Pins for the oracle's low-storage RK(5,4) (reading C13) and
for the time-dependent behaviour of the whole oracle (exact translation)."""
import math

import numpy as np
import pytest

from oracle import capi, dense, lsrk


def test_order_conditions():
    a, b, c = lsrk.butcher()
    res = lsrk.order_conditions(a, b, c)
    assert np.max(np.abs(res)) < 1e-15 * 8
    # c_s stored by the oracle equal the tableau row sums
    _, _, C = lsrk.coefficients()
    assert np.max(np.abs(C - c)) < 1e-15
    # A_1 = 0 makes the initial dU irrelevant
    A, _, _ = lsrk.coefficients()
    assert A[0] == 0.0


def test_stability_polynomial():
    g = lsrk.stability_polynomial()
    assert len(g) == 6
    assert np.max(np.abs(g[:5] - [1, 1, 0.5, 1 / 6, 1 / 24])) < 1e-15
    assert 0.004 < g[5] < 0.006  # gamma_5 ~ 0.005


def test_scalar_ode_order_four():
    # S:511 / S:694: y' = -y, observed order 4.0 +- 0.1
    errs = []
    for nsteps in (10, 20, 40, 80):
        dt = 1.0 / nsteps
        y = np.array([1.0])
        for _ in range(nsteps):
            y = lsrk.step(lambda u, t: -u, y, 0.0, dt)
        errs.append(abs(y[0] - math.exp(-1.0)))
    orders = [math.log2(errs[i] / errs[i + 1]) for i in range(3)]
    assert all(abs(o - 4.0) < 0.1 for o in orders[1:]), orders


def test_rk_step_is_stability_polynomial_of_operator():
    # On a linear operator L = M^-1 A (O1 dense), one oracle step equals sum_j gamma_j (dt L)^j u.
    from test_oracle_operator import tiny_spec
    spec = tiny_spec(2, 2, True)
    A, M = dense.assemble(spec)
    L = np.linalg.solve(M, A)
    N = L.shape[0]
    u = np.random.default_rng(11).uniform(-1, 1, N)
    dt = 0.01
    g = lsrk.stability_polynomial()
    exp = np.zeros(N)
    term = u.copy()
    for j in range(6):
        exp += g[j] * term
        term = dt * (L @ term)
    got = capi.rk_steps(spec, u, 0.0, dt, 1)
    assert np.max(np.abs(got - exp)) < 1e-13 * np.max(np.abs(exp))
    # and it approximates the semi-discrete exact solution exp(dt L) u with a local
    # error O(dt^5): halving dt divides the one-step error by ~32
    from scipy.linalg import expm
    e = []
    for h in (2e-3, 1e-3):
        e.append(np.max(np.abs(capi.rk_steps(spec, u, 0.0, h, 1) - expm(h * L) @ u)))
    assert 26.0 < e[0] / e[1] < 38.0, e


@pytest.mark.parametrize("k", [1, 2])
def test_convergence_exact_translation(k):
    # S:369 / S:688: L2 error vs the exact translated solution, order k+1 +- 0.25
    a = (1.0, 0.5)
    T = 0.25
    errs = []
    x, w = np.polynomial.legendre.leggauss(k + 1)
    x, w = 0.5 * (x + 1), 0.5 * w
    for nc in (4, 8, 16):
        spec = dict(d_x=1, d_v=1, k=k, cells=[nc, nc], lo=[0, 0], hi=[1, 1], a_const=list(a),
                    a_lin=[[0, 0], [0, 0]], flux="upwind")
        h = 1.0 / nc
        # nodal coordinates in global order (cell c1 slow, c0; node m1, m0 fastest)
        c1, c0, m1, m0 = np.meshgrid(np.arange(nc), np.arange(nc), np.arange(k + 1), np.arange(k + 1),
                                     indexing="ij")
        X = (c0 + x[m0]) * h
        Y = (c1 + x[m1]) * h
        W = w[m0] * w[m1] * h * h

        def f(X, Y):
            return np.sin(2 * np.pi * X) * np.sin(2 * np.pi * Y)

        u0 = f(X, Y).reshape(-1)
        dt = 0.05 / ((k + 1) ** 2 * (a[0] + a[1]) / h)
        nsteps = int(math.ceil(T / dt))
        dt = T / nsteps
        uT = capi.rk_steps(spec, u0, 0.0, dt, nsteps)
        ex = f(X - a[0] * T, Y - a[1] * T).reshape(-1)
        errs.append(math.sqrt(np.sum(W.reshape(-1) * (uT - ex) ** 2)))
    orders = [math.log2(errs[i] / errs[i + 1]) for i in range(2)]
    assert abs(orders[-1] - (k + 1)) < 0.25, (errs, orders)
