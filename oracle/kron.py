"""O3 oracle tier: the merged operator M^-1 A as a sum of 1D DG operators.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

P:776-843 splits the phase-space weak form into per-dimension cell and face terms
(block-diagonal Jacobian, n.a = n_x.a_x on x-faces and n_v.a_v on v-faces). With a
Cartesian mesh, the collocated diagonal mass and a field whose i-th component does
not depend on z_i (a_lin[i][i] = 0), M^-1 A acts along each dimension as an
independent 1D DG advection operator scaled pointwise by a_i(z):

    (M^-1 A u) = sum_i  |a_i(z)| * L1D_i(sign a_i)  applied along axis i        (upwind)
    (M^-1 A u) = sum_i  a_i(z)   * L1D_i(central)   applied along axis i        (central)

where L1D_i(s) is the merged 1D DG operator for unit speed s on the periodic line of
cells_i cells of width h_i. It is built here from the 1D weak form with explicit face
fluxes (not from any folded matrix), i.e.
    (A1 u)_{e,m} = sum_q h w_q (1/h) l_m'(xi_q) s u_{e,q}
                   - l_m(1) F_{e+1/2} + l_m(0) F_{e-1/2},   F = numerical flux
    L1D = diag(h w)^-1 A1.
Nodes and weights come from ``numpy.polynomial.legendre.leggauss``.
"""
from __future__ import annotations

import numpy as np


def _gl01(n):
    x, w = np.polynomial.legendre.leggauss(n)
    return 0.5 * (x + 1.0), 0.5 * w


def _lagrange(nodes, t):
    n = len(nodes)
    val = np.ones(n)
    der = np.zeros(n)
    for m in range(n):
        others = [k for k in range(n) if k != m]
        den = np.prod([nodes[m] - nodes[k] for k in others]) if others else 1.0
        val[m] = np.prod([t - nodes[k] for k in others]) / den if others else 1.0
        s = 0.0
        for l in others:
            rest = [k for k in others if k != l]
            s += (np.prod([t - nodes[k] for k in rest]) if rest else 1.0) / den
        der[m] = s
    return val, der


def op1d(n: int, ncells: int, h: float, speed: float, flux: str = "upwind") -> np.ndarray:
    """Merged 1D operator (size ncells*n) for constant speed on a periodic line."""
    x, w = _gl01(n)
    l0, _ = _lagrange(x, 0.0)
    l1, _ = _lagrange(x, 1.0)
    D = np.zeros((n, n))  # D[m, q] = l_m'(xi_q)
    for q in range(n):
        _, der = _lagrange(x, x[q])
        D[:, q] = der
    N = ncells * n
    A = np.zeros((N, N))
    for e in range(ncells):
        r = slice(e * n, (e + 1) * n)
        # cell term: sum_q h w_q (1/h) l_m'(xi_q) speed u_q
        A[r, r] += D * (w[None, :] * speed)
        # face at x = 1 of cell e (normal +1) and at x = 0 (normal -1): flux F(u-, u+, a.n)
        for side in (0, 1):
            en = (e + (1 if side else -1)) % ncells
            rn = slice(en * n, (en + 1) * n)
            lm = l1 if side else l0
            lp = l0 if side else l1
            an = speed if side else -speed
            if flux == "central":
                cm, cp = 0.5 * an, 0.5 * an
            else:
                cm = an if an > 0 else 0.0
                cp = 0.0 if an > 0 else an
            # F = cm * u- + cp * u+ ; contribution -l_m(face) F
            A[r, r] -= np.outer(lm, lm) * cm
            A[r, rn] -= np.outer(lm, lp) * cp
    Mdiag = np.tile(h * w, ncells)
    return A / Mdiag[:, None]


def _node_coords(spec):
    d = spec["d_x"] + spec["d_v"]
    n = spec["k"] + 1
    cells = [int(c) for c in spec["cells"]]
    lo = np.array(spec["lo"], float)
    h = (np.array(spec["hi"], float) - lo) / np.array(cells, float)
    x, _ = _gl01(n)
    # array axes: (c_{d-1}, ..., c_0, m_{d-1}, ..., m_0) -> C-order flattening = reading C19 order
    shape = [cells[i] for i in reversed(range(d))] + [n] * d
    Z = []
    for i in range(d):
        zc = lo[i] + (np.arange(cells[i])[:, None] + x[None, :]) * h[i]  # [cells_i, n]
        Z.append(np.broadcast_to(_place(zc, d, i, cells[i], n), shape))
    return Z, shape, h


def _place(zc, d, i, ci, n):
    """Reshape a [cells_i, n] table to broadcast over (c_{d-1..0}, m_{d-1..0})."""
    sh = [1] * (2 * d)
    sh[d - 1 - i] = ci
    sh[2 * d - 1 - i] = n
    # zc axes are (cell, node); the target keeps that relative order (cell axis first)
    return zc.reshape(sh)


def apply_merged(spec: dict, u: np.ndarray) -> np.ndarray:
    """M^-1 A(u) by the Kronecker-sum form (all configs small enough for numpy)."""
    d = spec["d_x"] + spec["d_v"]
    n = spec["k"] + 1
    cells = [int(c) for c in spec["cells"]]
    flux = spec.get("flux", "upwind")
    Z, shape, h = _node_coords(spec)
    U = u.reshape(shape)
    out = np.zeros(shape)
    lin = spec.get("a_lin")
    for i in range(d):
        a = np.full(shape, float(spec["a_const"][i]))
        if lin is not None:
            for j in range(d):
                if lin[i][j] != 0.0:
                    a = a + lin[i][j] * Z[j]
        ca, ma = d - 1 - i, 2 * d - 1 - i  # cell axis and node axis of dim i

        def along(L):
            # contract global 1D index (c_i, m_i) with L
            V = np.moveaxis(U, (ca, ma), (0, 1))
            sh = V.shape
            V2 = V.reshape(cells[i] * n, -1)
            R = (L @ V2).reshape(sh)
            return np.moveaxis(R, (0, 1), (ca, ma))

        if flux == "central":
            out += a * along(op1d(n, cells[i], h[i], 1.0, "central"))
        else:
            pos = along(op1d(n, cells[i], h[i], 1.0, "upwind"))
            neg = along(op1d(n, cells[i], h[i], -1.0, "upwind"))
            out += np.where(a > 0, a * pos, -a * neg)
    return out.reshape(-1)
