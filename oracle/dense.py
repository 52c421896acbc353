"""O1 oracle tier: brute-force dense assembly of the DG advection operator.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Definition followed (Eq. into:adv:ref; sign P:236; readings C2-C5):
    M_ij = int_cell phi_i phi_j |J|
    A_ij = int_cell grad(phi_i) . a phi_j |J|  -  sum_faces int_face phi_i (a.n) phi_j^{up} |J_face|
with the numerical flux of S:387-395 evaluated pointwise at face quadrature points.
Integrals use an OVER-INTEGRATED tensor Gauss rule with n+2 points per dimension,
taken from ``numpy.polynomial.legendre.leggauss`` (independent of the O2 Newton
iteration), so the claim that the n-point collocated rule is exact is tested, not
assumed (SURVEY 8(c) "O1"). The basis nodes also come from ``leggauss``.
Only for tiny meshes (global DoF count <= ~4096).
"""
from __future__ import annotations

import itertools
from functools import reduce

import numpy as np


def _gl01(n: int):
    x, w = np.polynomial.legendre.leggauss(n)
    return 0.5 * (x + 1.0), 0.5 * w


def _lagrange_matrix(nodes: np.ndarray, pts: np.ndarray):
    """B[q, m] = l_m(pts_q), G[q, m] = l_m'(pts_q) for the Lagrange basis on nodes."""
    n = len(nodes)
    B = np.ones((len(pts), n))
    G = np.zeros((len(pts), n))
    for m in range(n):
        others = [k for k in range(n) if k != m]
        den = np.prod([nodes[m] - nodes[k] for k in others]) if others else 1.0
        B[:, m] = np.prod([pts - nodes[k] for k in others], axis=0) / den if others else 1.0
        for l in others:
            rest = [k for k in others if k != l]
            G[:, m] += (np.prod([pts - nodes[k] for k in rest], axis=0) if rest else 1.0) / den
    return B, G


def _kron_list(mats):
    """Tensor product with dim 0 fastest: kron(M_{d-1}, ..., M_0)."""
    return reduce(np.kron, list(reversed(mats)))


def _speed(spec, i, Z):
    d = spec["d_x"] + spec["d_v"]
    a = np.full(Z[0].shape, float(spec["a_const"][i]))
    lin = spec.get("a_lin")
    if lin is not None:
        for j in range(d):
            if lin[i][j] != 0.0:
                a = a + lin[i][j] * Z[j]
    return a


def assemble(spec: dict, over: int = 2, nodes=None):
    """Return dense (A, M) in global DoF order (reading C19). ``nodes``: the 1D interpolation nodes on
    [0, 1] of the nodal basis (default: the n Gauss points, reading C1; oracle/gll.py passes the
    Gauss-Lobatto points of the paper's default basis)."""
    d = spec["d_x"] + spec["d_v"]
    n = spec["k"] + 1
    cells = [int(c) for c in spec["cells"]]
    lo = np.array(spec["lo"], float)
    h = (np.array(spec["hi"], float) - lo) / np.array(cells, float)
    nd = n ** d
    ncell = int(np.prod(cells))
    N = ncell * nd
    flux = spec.get("flux", "upwind")
    if nodes is None:
        nodes, _ = _gl01(n)
    nodes = np.asarray(nodes, float)
    assert nodes.shape == (n,)
    xq, wq = _gl01(n + over)
    B, G = _lagrange_matrix(nodes, xq)           # [nq, n]
    b0, _ = _lagrange_matrix(nodes, np.array([0.0]))
    b1, _ = _lagrange_matrix(nodes, np.array([1.0]))
    Jdet = float(np.prod(h))
    A = np.zeros((N, N))
    M = np.zeros((N, N))
    strides = [int(np.prod(cells[:i])) for i in range(d)]

    def cell_id(c):
        return sum(int(c[i]) * strides[i] for i in range(d))

    Wcell = _kron_list([wq] * d)
    Phi = _kron_list([B] * d)                     # [nq^d, nd]
    dPhi = [_kron_list([G / h[i] if j == i else B for j in range(d)]) for i in range(d)]
    for c in itertools.product(*[range(ci) for ci in cells]):
        g = cell_id(c)
        rows = slice(g * nd, (g + 1) * nd)
        # physical coordinates of the over-integration points, per dim, broadcast to the d-dim grid
        z1d = [lo[i] + (c[i] + xq) * h[i] for i in range(d)]
        Z = [_kron_list([z1d[j] if j == i else np.ones(len(xq)) for j in range(d)]) for i in range(d)]
        M[rows, rows] += Phi.T @ (Wcell[:, None] * Jdet * Phi)
        for i in range(d):
            ai = _speed(spec, i, Z)
            A[rows, rows] += dPhi[i].T @ ((Wcell * Jdet * ai)[:, None] * Phi)
        # faces
        for i in range(d):
            Jf = Jdet / h[i]
            for side in (0, 1):
                own_row = b1 if side else b0             # phi_m at own face (xi_i = side)
                nb_row = b0 if side else b1              # phi_p^nb at the shared face
                cn = list(c)
                cn[i] = (c[i] + (1 if side else -1)) % cells[i]
                gn = cell_id(cn)
                cols_nb = slice(gn * nd, (gn + 1) * nd)
                Wf = _kron_list([wq if j != i else np.ones(1) for j in range(d)])
                Phi_own = _kron_list([B if j != i else own_row for j in range(d)])
                Phi_nb = _kron_list([B if j != i else nb_row for j in range(d)])
                zf = [np.full(1, lo[i] + (c[i] + side) * h[i]) if j == i else z1d[j] for j in range(d)]
                Zf = [_kron_list([zf[j] if j == l else np.ones(len(zf[j])) for j in range(d)]) for l in range(d)]
                an = (1.0 if side else -1.0) * _speed(spec, i, Zf)
                if flux == "central":
                    w_own = 0.5 * an
                    w_nb = 0.5 * an
                else:
                    w_own = np.where(an > 0, an, 0.0)
                    w_nb = np.where(an > 0, 0.0, an)
                A[rows, rows] -= Phi_own.T @ ((Wf * Jf * w_own)[:, None] * Phi_own)
                A[rows, cols_nb] -= Phi_own.T @ ((Wf * Jf * w_nb)[:, None] * Phi_nb)
    return A, M


def apply_advection(spec: dict, u: np.ndarray, merged: bool = False) -> np.ndarray:
    A, M = assemble(spec)
    v = A @ u
    return np.linalg.solve(M, v) if merged else v
