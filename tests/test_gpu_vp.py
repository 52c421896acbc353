"""GPU parity of the Vlasov-Poisson path: hd_vp_fields,
hd_apply_advection_vp and hd_vp_rk_step against the oracle (oracle/vp.py), and the Landau-damping run
against the dispersion-relation root (the paper's own verification P:4008-4009)."""
import numpy as np
import pytest

from oracle import capi
from oracle import vp

from test_gpu_parity import assert_close, dev, host, mesh
from test_oracle_vp import vp_spec

pytestmark = pytest.mark.gpu

SPECS = [
    ("1x1v", vp_spec(1, 3, [6, 4], [4 * np.pi], 3.0)),
    ("1x1v-k4", vp_spec(1, 4, [5, 2], [2.0], 1.0)),
    ("2x2v", vp_spec(2, 1, [3, 4, 2, 2], [2.0, 3.0], 1.5)),
    ("2x2v-k2", vp_spec(2, 2, [3, 3, 2, 2], [1.0, 1.0], 2.0)),
    ("3x3v", vp_spec(3, 1, [3, 3, 2, 2, 2, 2], [1.0, 2.0, 1.5], 1.0)),
]


def _f(spec, seed):
    return 0.5 + 0.3 * np.random.default_rng(seed).uniform(-1, 1, capi.dof_count(spec))


@pytest.mark.parametrize("name,spec", SPECS, ids=[s[0] for s in SPECS])
def test_vp_fields(name, spec):
    import torch
    m = mesh(spec)
    f = _f(spec, 1)
    nxn, ne = m.vp_sizes()
    rho = torch.empty(nxn, dtype=torch.float64, device="cuda")
    E = torch.empty(ne, dtype=torch.float64, device="cuda")
    m.vp_fields(dev(f), rho, E)
    r_ref = vp.density(spec, f)
    assert_close(host(rho), r_ref.reshape(-1), 1e-12, name + " rho")
    E_ref = vp.efield(spec, r_ref)
    if np.max(np.abs(E_ref)) > 0:
        assert_close(host(E), E_ref.reshape(-1), 1e-12, name + " E")


@pytest.mark.parametrize("flux", ["upwind", "central"])
@pytest.mark.parametrize("name,spec", SPECS, ids=[s[0] for s in SPECS])
def test_vp_apply(name, spec, flux):
    """v <- A(u) with a = (v, -E(x)), E changing sign inside cells."""
    import torch
    spec = dict(spec, flux=flux)
    m = mesh(spec)
    N = m.owned_dofs
    X, _ = vp.x_nodes(spec)
    E = np.stack([0.7 * np.sin(2 * np.pi * X[..., i] / (spec["hi"][i] - spec["lo"][i]) + 0.3 * i) + 0.05
                  for i in range(spec["d_x"])])
    u = np.random.default_rng(2).uniform(-1, 1, N)
    v = torch.full((N,), float("nan"), dtype=torch.float64, device="cuda")
    m.apply_advection_vp(dev(u), dev(E.reshape(-1)), v)
    assert_close(host(v), vp.apply_advection_vp(spec, u, E), 1e-12, name + " A_vp")


@pytest.mark.parametrize("name,spec", SPECS[:3], ids=[s[0] for s in SPECS[:3]])
def test_vp_rk10(name, spec):
    """Ten coupled steps (E recomputed from every stage's f) against the oracle, <= 1e-10."""
    import torch
    m = mesh(spec)
    f = _f(spec, 4)
    dt = 0.02
    bufs = [dev(f), torch.empty(m.owned_dofs, dtype=torch.float64, device="cuda"),
            torch.empty(m.owned_dofs, dtype=torch.float64, device="cuda")]
    m.vp_rk_step(bufs, 0.0, dt, 10)
    ref = vp.rk_steps(spec, f, dt, 10)
    assert_close(host(bufs[0]), ref, 1e-10, name + " vp rk10")


def test_landau_damping():
    """Weak Landau damping, 1x1v, kappa = 0.5, alpha = 0.01, v in [-6, 6]: the field energy
    1/2 int E^2 decays at 2 gamma and oscillates at 2 omega_r of the dispersion root, both within 5%; total
    mass conserved."""
    import torch
    kap, alpha = 0.5, 0.01
    spec = vp_spec(1, 3, [16, 32], [2 * np.pi / kap], 6.0)
    m = mesh(spec)
    n = 4
    xi, _ = capi.gauss_legendre(n)
    cx, cv = spec["cells"]
    hx, hv = 2 * np.pi / kap / cx, 12.0 / cv
    X = ((np.arange(cx)[:, None] + xi[None, :]) * hx)             # [cx, jx]
    V = (-6.0 + (np.arange(cv)[:, None] + xi[None, :]) * hv)     # [cv, jv]
    f0 = ((1 + alpha * np.cos(kap * X))[None, :, None, :] *
          (np.exp(-V**2 / 2) / np.sqrt(2 * np.pi))[:, None, :, None]).reshape(-1)  # [cv, cx, jv, jx]
    N = m.owned_dofs
    assert f0.size == N
    bufs = [dev(f0), torch.empty(N, dtype=torch.float64, device="cuda"),
            torch.empty(N, dtype=torch.float64, device="cuda")]
    nxn, ne = m.vp_sizes()
    E = torch.empty(ne, dtype=torch.float64, device="cuda")
    dt, every, T = 0.01, 5, 20.0
    ts, en = [], []
    ones = np.ones(N)
    mass0 = capi.apply_mass(spec, ones) @ f0
    t = 0.0
    while t < T - 1e-9:
        m.vp_fields(bufs[0], None, E)
        ts.append(t)
        en.append(vp.field_energy(spec, host(E)))
        m.vp_rk_step(bufs, t, dt, every)
        t += dt * every
    ts, en = np.array(ts), np.array(en)
    assert np.all(np.isfinite(en))
    # local maxima of the energy after the initial transient
    pk = [i for i in range(1, len(en) - 1) if en[i] > en[i - 1] and en[i] >= en[i + 1] and ts[i] > 1.5]
    assert len(pk) >= 4, pk
    slope = np.polyfit(ts[pk], np.log(en[pk]), 1)[0]
    om = vp.landau_root(kap)
    assert abs(slope - 2 * om.imag) <= 0.05 * abs(2 * om.imag), (slope, 2 * om.imag)
    period = np.mean(np.diff(ts[pk]))           # energy oscillates at 2 omega_r
    assert abs(np.pi / period - om.real) <= 0.05 * om.real, (np.pi / period, om.real)
    mass = capi.apply_mass(spec, ones) @ host(bufs[0])
    assert abs(mass - mass0) <= 1e-10 * abs(mass0)
