"""Vlasov-Poisson oracle: density reduction, periodic Poisson / electric field, the
advection operator with the composed field a = (v, -E(x)), the coupled LSRK step and the Landau-damping
dispersion root.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``). Plain numpy, fp64, small meshes.

Passages followed:
  * P:3926-3963, Eq. equ:vp:close: f_t + v.grad_x f - E.grad_v f = 0, rho = 1 - int f dv, -lap phi = rho,
    E = -grad phi; the paper's five steps per stage (rho, Poisson RHS, solve, E, advect with a = (v, -E)).
  * a is composed on the fly from the x part (v, the v coordinate) and the v part (-E at x).
  * S:567-575 (SPEC substitute for the paper's multigrid, reading C24): a Fourier solve on the periodic x
    box. Here the Fourier coefficients of rho_h are its Gauss rule (the collocated quadrature of the DG
    space): rhohat(m) = |Omega_x|^-1 sum_nodes W rho e^{-i k.x}, k_i = 2 pi m_i / L_i, |m_i| <= K_i =
    floor((cells_i - 1) / 2) (modes whose per-cell phase stays below pi, so the n-point rule of each cell does
    not alias them into each other), the zero mode dropped; phi = sum rhohat / |k|^2 e^{i k.x}.
  * Alg. 2 in collocation form (reading C1) for the operator, both traces and the S:387-395
    flux at every face point, the speed evaluated at the face point.
  * Landau damping, root of 1 + kappa^-2 (1 + zeta Z(zeta)) = 0, zeta = omega / (sqrt(2) kappa),
    Z(zeta) = i sqrt(pi) w(zeta) (Faddeeva function, scipy.special.wofz).
Layout (reading C19): cell g = c_x + |C_x| c_v, in-cell j = j_x + n^d_x j_v, x dims fastest.
"""
from __future__ import annotations

import itertools

import numpy as np

from . import capi, lsrk


def _geom(spec):
    d_x, d_v = spec["d_x"], spec["d_v"]
    d = d_x + d_v
    n = spec["k"] + 1
    cells = [int(c) for c in spec["cells"]]
    lo = np.array(spec["lo"], float)
    hi = np.array(spec["hi"], float)
    h = (hi - lo) / np.array(cells, float)
    xi, w = capi.gauss_legendre(n)
    return d_x, d_v, d, n, cells, lo, hi, h, xi, w


def _multi(n, dims):
    """multi-indices of n^dims nodes, first index fastest: array [n^dims, dims]"""
    return np.array([list(reversed(t)) for t in itertools.product(range(n), repeat=dims)], dtype=int).reshape(-1, dims)


def x_nodes(spec):
    """Coordinates X[cx, jx, i] and Gauss weights W[cx, jx] (with |J_x|) of every x node."""
    d_x, d_v, d, n, cells, lo, hi, h, xi, w = _geom(spec)
    cm = _multi_cells(cells[:d_x])
    jm = _multi(n, d_x)
    X = lo[:d_x][None, None, :] + (cm[:, None, :] + xi[jm][None, :, :]) * h[:d_x][None, None, :]
    W = np.prod(w[jm], axis=1)[None, :] * np.prod(h[:d_x]) * np.ones((len(cm), 1))
    return X, W


def _multi_cells(cells):
    out = []
    for g in range(int(np.prod(cells))):
        c, r = [], g
        for L in cells:
            c.append(r % L)
            r //= L
        out.append(c)
    return np.array(out, dtype=float).reshape(-1, len(cells))


def density(spec, f):
    """rho[cx, jx] = 1 - sum_{v cells, v nodes} f |J_v| prod w."""
    d_x, d_v, d, n, cells, lo, hi, h, xi, w = _geom(spec)
    ncx = int(np.prod(cells[:d_x]))
    ncv = int(np.prod(cells[d_x:]))
    nx, nv = n ** d_x, n ** d_v
    f4 = np.asarray(f, float).reshape(ncv, ncx, nv, nx)
    wv = np.prod(w[_multi(n, d_v)], axis=1) * np.prod(h[d_x:])
    return 1.0 - np.einsum("vcjx,j->cx", f4, wv)


def modes(spec):
    d_x, d_v, d, n, cells, lo, hi, h, xi, w = _geom(spec)
    K = [(cells[i] - 1) // 2 for i in range(d_x)]
    ms = np.array(list(itertools.product(*[range(-K[i], K[i] + 1) for i in range(d_x)])), dtype=float)
    L = hi[:d_x] - lo[:d_x]
    return 2.0 * np.pi * ms / L[None, :]


def rho_hat(spec, rho):
    """Fourier coefficients of rho_h by its Gauss rule, per mode of ``modes(spec)``."""
    d_x = spec["d_x"]
    X, W = x_nodes(spec)
    kv = modes(spec)
    vol = float(np.prod(np.array(spec["hi"][:d_x]) - np.array(spec["lo"][:d_x])))
    ph = np.einsum("mi,cji->mcj", kv, X)
    return np.einsum("mcj,cj->m", np.exp(-1j * ph), W * rho) / vol


def phi_at(spec, rho, x):
    """phi(x) = sum_{m != 0} rhohat / |k|^2 e^{i k.x} at points x[p, i] (solves -lap phi = rho mode by mode)."""
    kv = modes(spec)
    k2 = np.sum(kv * kv, axis=1)
    rh = rho_hat(spec, rho)
    keep = k2 > 0
    return np.real(np.exp(1j * (np.asarray(x) @ kv[keep].T)) @ (rh[keep] / k2[keep]))


def efield(spec, rho):
    """E = -grad phi at every x node: E[i, cx, jx] = Re sum_{m != 0} (-i k_i) rhohat / |k|^2 e^{i k.x}."""
    d_x = spec["d_x"]
    X, _ = x_nodes(spec)
    kv = modes(spec)
    k2 = np.sum(kv * kv, axis=1)
    rh = rho_hat(spec, rho)
    keep = k2 > 0
    ph = np.exp(1j * np.einsum("mi,cji->mcj", kv[keep], X))
    out = np.empty((d_x,) + X.shape[:2])
    for i in range(d_x):
        out[i] = np.real(np.einsum("m,mcj->cj", -1j * kv[keep, i] * rh[keep] / k2[keep], ph))
    return out


def apply_advection_vp(spec, u, E):
    """v = A(u), weak form, a = (a_const + a_lin z) - (0, E(x)) -- Alg. 2 in collocation form, cell by cell."""
    d_x, d_v, d, n, cells, lo, hi, h, xi, w = _geom(spec)
    flux = spec.get("flux", "upwind")
    a_const = np.array(spec["a_const"], float)
    a_lin = np.array(spec.get("a_lin", np.zeros((d, d))), float)
    E = np.asarray(E, float).reshape(d_x, -1, n ** d_x)
    nd = n ** d
    nx = n ** d_x
    ncx = int(np.prod(cells[:d_x]))
    Jdet = float(np.prod(h))
    M = _multi(n, d)                                  # [nd, d]
    W = np.prod(w[M], axis=1)
    l0, _ = capi.lagrange_eval(n, 0.0)
    l1, _ = capi.lagrange_eval(n, 1.0)
    D = np.array([capi.lagrange_eval(n, xi[q])[1] for q in range(n)])  # D[q, m] = l_m'(xi_q)
    pw = [n ** i for i in range(d)]
    jx_of = (M[:, :d_x] * np.array(pw[:d_x])).sum(axis=1)
    cm = _multi_cells(cells).astype(int)
    strides = [int(np.prod(cells[:i])) for i in range(d)]
    u = np.asarray(u, float).reshape(-1, nd)
    out = np.zeros_like(u)

    def speed(i, z, cx, jx):
        a = a_const[i] + z @ a_lin[i]
        if i >= d_x:
            a = a - E[i - d_x, cx, jx]
        return a

    for g in range(len(cm)):
        c = cm[g]
        cx = g % ncx
        z = lo[None, :] + (c[None, :] + xi[M]) * h[None, :]  # [nd, d]
        b = np.zeros(nd)
        for i in range(d):
            t = speed(i, z, cx, jx_of) / h[i] * Jdet * W * u[g]      # t_q (Alg. 2 step 2)
            for m in range(nd):                                        # test with l'_{m_i}(xi_q)
                base = m - M[m, i] * pw[i]
                b[m] += sum(D[q, M[m, i]] * t[base + q * pw[i]] for q in range(n))
        for i in range(d):
            Jf = Jdet / h[i]
            for side in (0, 1):
                cn = c.copy()
                cn[i] = (c[i] + (1 if side else -1)) % cells[i]
                un = u[int(np.dot(cn, strides))]
                lm, lp = (l1, l0) if side else (l0, l1)
                for m in np.nonzero(M[:, i] == 0)[0]:
                    line = m + np.arange(n) * pw[i]
                    um = float(lm @ u[g][line])
                    up = float(lp @ un[line])
                    zf = z[m].copy()
                    zf[i] = lo[i] + (c[i] + side) * h[i]
                    wf = np.prod([w[M[m, j]] for j in range(d) if j != i])
                    an = (1.0 if side else -1.0) * float(speed(i, zf, cx, jx_of[m]))
                    F = 0.5 * an * (um + up) + (0.0 if flux == "central" else 0.5 * abs(an) * (um - up))
                    b[line] -= lm * wf * Jf * F
        out[g] = b
    return out.reshape(-1)


def mass_inverse(spec, v):
    return capi.apply_inv_mass(spec, v)


def rhs(spec, f):
    """M^-1 A(f; E(f)): the five steps of one stage."""
    E = efield(spec, density(spec, f))
    return mass_inverse(spec, apply_advection_vp(spec, f, E))


def rk_steps(spec, f, dt, nsteps):
    u = np.array(f, float)
    for _ in range(nsteps):
        u = lsrk.step(lambda x, t: rhs(spec, x), u, 0.0, dt)
    return u


def field_energy(spec, E):
    """1/2 int |E|^2 dx by the Gauss rule of the x nodes."""
    _, W = x_nodes(spec)
    return 0.5 * float(np.sum(W[None] * np.asarray(E).reshape((spec["d_x"],) + W.shape) ** 2))


def landau_root(kappa, omega0=1.4 - 0.15j, tol=1e-14):
    """Root of the linear Landau dispersion relation eps(omega) = 1 + kappa^-2 (1 + zeta Z(zeta)),
    zeta = omega / (sqrt(2) kappa), by the secant method."""
    from scipy.special import wofz

    def eps(om):
        zeta = om / (np.sqrt(2.0) * kappa)
        Z = 1j * np.sqrt(np.pi) * wofz(zeta)
        return 1.0 + (1.0 + zeta * Z) / kappa**2

    x0, x1 = omega0, omega0 * (1 + 1e-3)
    f0, f1 = eps(x0), eps(x1)
    for _ in range(100):
        x2 = x1 - f1 * (x1 - x0) / (f1 - f0)
        if abs(x2 - x1) < tol:
            return x2
        x0, f0, x1, f1 = x1, f1, x2, eps(x2)
    return x1
