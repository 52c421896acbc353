"""Pins of the Vlasov-Poisson oracle (oracle/vp.py) against closed forms, special cases
that reduce to the pinned O2 operator, invariants and a textbook dispersion root. CPU only."""
import numpy as np
import pytest

from oracle import capi
from oracle import vp


def vp_spec(d_x, k, cells, L, vmax, flux="upwind", a_v=None):
    d = 2 * d_x
    lin = [[0.0] * d for _ in range(d)]
    for i in range(d_x):
        lin[i][d_x + i] = 1.0
    return dict(d_x=d_x, d_v=d_x, k=k, cells=list(cells), lo=[0.0] * d_x + [-vmax] * d_x,
                hi=list(L) + [vmax] * d_x, a_const=[0.0] * d_x + list(a_v or [0.0] * d_x), a_lin=lin, flux=flux)


S2 = vp_spec(1, 3, [6, 4], [4 * np.pi], 3.0)
S4 = vp_spec(2, 1, [3, 2, 2, 2], [2.0, 3.0], 1.5)


def test_density_constant_and_separable():
    """f = c gives rho = 1 - c |Omega_v|; f = g(x) h(v) with h of degree <= 2k+1 per v dim (integrated exactly
    by the Gauss rule) gives rho = 1 - g(x) int h dv."""
    for spec in (S2, S4):
        N = capi.dof_count(spec)
        vol_v = np.prod([spec["hi"][i] - spec["lo"][i] for i in range(spec["d_x"], 2 * spec["d_x"])])
        rho = vp.density(spec, np.full(N, 0.25))
        assert np.allclose(rho, 1 - 0.25 * vol_v, rtol=0, atol=1e-14)
    # separable, 1x1v: g(x) = cos(x / 2), h(v) = v^2 + v^7 (degree 7 = 2k+1 for k = 3): int_{-3}^{3} h = 18
    spec = S2
    n, cells = spec["k"] + 1, spec["cells"]
    xi, _ = capi.gauss_legendre(n)
    hx = (spec["hi"][0] - spec["lo"][0]) / cells[0]
    hv = (spec["hi"][1] - spec["lo"][1]) / cells[1]
    f = np.empty(capi.dof_count(spec))
    for cv in range(cells[1]):
        for cx in range(cells[0]):
            for jv in range(n):
                for jx in range(n):
                    x = (cx + xi[jx]) * hx
                    v = spec["lo"][1] + (cv + xi[jv]) * hv
                    f[(cv * cells[0] + cx) * n * n + jv * n + jx] = np.cos(x / 2) * (v**2 + v**7)
    rho = vp.density(spec, f)
    X, _ = vp.x_nodes(spec)
    assert np.allclose(rho, 1 - np.cos(X[..., 0] / 2) * 18.0, rtol=0, atol=1e-12)


def test_poisson_single_modes():
    """-phi'' = sin(kappa x) gives E = -phi' = -cos(kappa x) / kappa; in 2D x a mode along y only,
    rho = cos(kappa_y y), gives E = (0, sin(kappa_y y) / kappa_y). The retained modes keep their per-cell
    phase below pi, where the n-point Gauss rule of the nodal samples is exact to round-off for these
    modes."""
    spec = vp_spec(1, 3, [32, 2], [4 * np.pi], 3.0)
    X, _ = vp.x_nodes(spec)
    kap = 0.5
    E = vp.efield(spec, np.sin(kap * X[..., 0]))
    assert np.max(np.abs(E[0] + np.cos(kap * X[..., 0]) / kap)) <= 1e-12
    spec2 = vp_spec(2, 2, [4, 16, 2, 2], [1.0, 2 * np.pi], 2.0)
    X2, _ = vp.x_nodes(spec2)
    E2 = vp.efield(spec2, np.cos(X2[..., 1]))
    assert np.max(np.abs(E2[0])) <= 1e-10
    assert np.max(np.abs(E2[1] - np.sin(X2[..., 1]))) <= 1e-12
    # rho constant: no field
    assert np.max(np.abs(vp.efield(spec2, np.full(X2.shape[:2], 0.7)))) <= 1e-13


def test_efield_is_minus_gradient_of_phi():
    """E = -grad phi (central differences of the oracle's phi at the x nodes), random rho, 2D x."""
    spec = vp_spec(2, 1, [3, 4, 2, 2], [1.0, 1.5], 1.0)
    X, _ = vp.x_nodes(spec)
    rho = np.random.default_rng(3).uniform(-1, 1, X.shape[:2])
    E = vp.efield(spec, rho)
    pts = X.reshape(-1, 2)
    dlt = 1e-5
    for i in range(2):
        e = np.zeros(2)
        e[i] = dlt
        fd = -(vp.phi_at(spec, rho, pts + e) - vp.phi_at(spec, rho, pts - e)) / (2 * dlt)
        assert np.max(np.abs(fd - E[i].reshape(-1))) <= 1e-6 * np.max(np.abs(E[i]))


@pytest.mark.parametrize("spec", [S2, S4], ids=["1x1v", "2x2v"])
def test_vp_operator_reduces_to_o2(spec):
    """E = 0 gives the O2 operator with a = (v, 0); E = constant E0 gives O2 with a_v = -E0 (pinned tiers)."""
    N = capi.dof_count(spec)
    u = np.random.default_rng(11).uniform(-1, 1, N)
    d_x, n = spec["d_x"], spec["k"] + 1
    ncx = int(np.prod(spec["cells"][:d_x]))
    E0 = np.zeros((d_x, ncx, n ** d_x))
    got = vp.apply_advection_vp(spec, u, E0)
    ref = capi.apply_advection(spec, u)
    assert np.max(np.abs(got - ref)) <= 1e-13 * np.max(np.abs(ref))
    Ec = [0.4, -0.3][:d_x]
    E1 = np.stack([np.full((ncx, n ** d_x), e) for e in Ec])
    got = vp.apply_advection_vp(spec, u, E1)
    ref = capi.apply_advection(dict(spec, a_const=[0.0] * d_x + [-e for e in Ec]), u)
    assert np.max(np.abs(got - ref)) <= 1e-13 * np.max(np.abs(ref))


@pytest.mark.parametrize("flux", ["upwind", "central"])
def test_vp_operator_invariants(flux):
    """Varying E(x) whose sign changes inside cells: total mass conserved (sum of the weak form = 0),
    a constant state is steady (div a = 0), and the upwind operator dissipates (u^T A u <= 0), the central
    one conserves u^T M u (u^T A u = 0)."""
    spec = dict(S2, flux=flux)
    N = capi.dof_count(spec)
    X, _ = vp.x_nodes(spec)
    E = (0.8 * np.sin(0.5 * X[..., 0]) + 0.1)[None]
    u = np.random.default_rng(5).uniform(-1, 1, N)
    v = vp.apply_advection_vp(spec, u, E)
    assert abs(v.sum()) <= 1e-12 * np.abs(v).sum()
    assert np.max(np.abs(vp.apply_advection_vp(spec, np.full(N, 0.3), E))) <= 1e-12
    q = float(u @ v)
    if flux == "central":
        assert abs(q) <= 1e-12 * np.abs(u).sum() * np.abs(v).max()
    else:
        assert q < 0


def test_landau_dispersion_root():
    """kappa = 0.5: omega = 1.4156 - 0.1533 i (the textbook linear Landau damping values)."""
    om = vp.landau_root(0.5)
    assert abs(om.real - 1.4156) < 5e-4 and abs(om.imag + 0.1533) < 5e-4
    assert abs(vp.landau_root(0.4).imag + 0.0661) < 5e-4   # weaker damping at longer wavelength


def test_vp_rk_conserves_mass():
    """Ten coupled LSRK steps (E recomputed per stage) conserve int f (weights sum) to round-off."""
    spec = S2
    N = capi.dof_count(spec)
    X, _ = vp.x_nodes(spec)
    rng = np.random.default_rng(8)
    f = 0.1 + 0.01 * rng.uniform(-1, 1, N)
    m0 = capi.apply_mass(spec, np.ones(N)) @ f
    g = vp.rk_steps(spec, f, 0.01, 10)
    assert abs(capi.apply_mass(spec, np.ones(N)) @ g - m0) <= 1e-12 * abs(m0)
    assert np.max(np.abs(g - f)) > 1e-6
