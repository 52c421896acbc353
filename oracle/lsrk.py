"""Low-storage RK(5,4) of the oracle, as numbers and as a Butcher tableau.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

P:3141-3145: "low-storage Runge--Kutta scheme of order 4 with 5 stages, which uses
two auxiliary vectors besides the solution vector [Kennedy00]". The paper prints no
coefficients (reading C13): the oracle uses the Williamson 2N form

    dU <- A_s dU + dt F(U);   U <- U + B_s dU,   s = 1..5,

with the Carpenter-Kennedy five-stage fourth-order 2N coefficients, which live in
``hd_oracle.cpp`` and are read back here through the C API so that the tests pin
exactly what the oracle integrates with.
"""
from __future__ import annotations

import numpy as np

from . import capi


def coefficients():
    return capi.rk_coefficients()


def butcher(A=None, B=None):
    """Butcher tableau (a, b, c) of the 2N scheme. Stage i is evaluated at U_{i-1}:
    U_s = U_0 + dt sum_j K_j sum_{r=j}^{s} B_r prod_{l=j+1}^{r} A_l."""
    if A is None:
        A, B, _ = coefficients()
    s = len(A)

    def coef(j, upto):
        tot = 0.0
        for r in range(j, upto + 1):
            p = 1.0
            for l in range(j + 1, r + 1):
                p *= A[l]
            tot += B[r] * p
        return tot

    a = np.zeros((s, s))
    for i in range(s):
        for j in range(i):
            a[i, j] = coef(j, i - 1)
    b = np.array([coef(j, s - 1) for j in range(s)])
    c = a.sum(axis=1)
    return a, b, c


def order_conditions(a, b, c):
    """Residuals of the 8 classical conditions for order 4."""
    return np.array([
        b.sum() - 1.0,
        b @ c - 1.0 / 2,
        b @ c**2 - 1.0 / 3,
        b @ (a @ c) - 1.0 / 6,
        b @ c**3 - 1.0 / 4,
        b @ (c * (a @ c)) - 1.0 / 8,
        b @ (a @ c**2) - 1.0 / 12,
        b @ (a @ (a @ c)) - 1.0 / 24,
    ])


def step(F, u, t, dt, A=None, B=None, C=None):
    """One 2N step for a callable F(u, t) on numpy arrays (plain loop)."""
    if A is None:
        A, B, C = coefficients()
    du = np.zeros_like(u)
    u = u.copy()
    for s in range(5):
        du = A[s] * du + dt * F(u, t + C[s] * dt)
        u = u + B[s] * du
    return u


def stability_polynomial(A=None, B=None):
    """Coefficients gamma_j of R(z) = sum_j gamma_j z^j, from the 2N recurrence applied to
    y' = lambda y with polynomial arithmetic in z = lambda dt."""
    if A is None:
        A, B, _ = coefficients()
    P = np.polynomial.polynomial
    u = np.array([1.0])
    du = np.array([0.0])
    for s in range(5):
        du = P.polyadd(A[s] * du, P.polymulx(u))
        u = P.polyadd(u, B[s] * du)
    return u
