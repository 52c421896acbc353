"""GPU parity of the GLL <-> Gauss basis change and of the operator / time loop in the GLL basis
(hd_basis_change, hd_apply_advection_gll, hd_rk_step_gll; SURVEY §8(f) NEXT-2 Cartesian part; P:228-233,
P:509-518) against oracle/gll.py. Bars as for the product operator (reading C17): <= 1e-12 per
application, <= 1e-10 after 10 RK steps; the basis change alone (d sweeps of an n x n matrix) <= 1e-13."""
import numpy as np
import pytest

from oracle import gll as ogll
from paper_2002_08110_b200 import configs, inputs

from test_gpu_parity import DEGENERATE, SMALL, TOL_APPLY, TOL_RK10, assert_close, dev, host, mesh, spec_of

pytestmark = pytest.mark.gpu

TOL_BASIS = 1e-13
CASES = SMALL + [(n, s) for n, s in DEGENERATE if s["k"] + 1 >= 2]


@pytest.mark.parametrize("name,spec", CASES, ids=[s[0] for s in CASES])
def test_basis_change_small_meshes(name, spec):
    """Every built (d, n), ragged cell batches, all four kinds, out of place and in place; T^-1 T = I."""
    import torch
    m = mesh(spec)
    N = m.owned_dofs
    u = np.random.default_rng(abs(hash(name)) % (2**32) + 11).uniform(-1, 1, N)
    ud = dev(u)
    for kind in ogll.KINDS:
        v = torch.full((N,), float("nan"), dtype=torch.float64, device="cuda")
        m.basis_change(ud, v, kind)
        assert_close(host(v), ogll.basis_change(spec, u, kind), TOL_BASIS, f"{name} {kind}")
        w = ud.clone()
        m.basis_change(w, w, kind)
        assert torch.equal(w, v), f"{name} {kind}: in place differs from out of place"
    w = ud.clone()
    m.basis_change(w, w, "gll_to_gauss")
    m.basis_change(w, w, "gauss_to_gll")
    assert_close(host(w), u, TOL_BASIS, name + " round trip")


@pytest.mark.parametrize("name,spec", CASES, ids=[s[0] for s in CASES])
def test_apply_advection_gll_small_meshes(name, spec):
    import torch
    m = mesh(spec)
    N = m.owned_dofs
    u = np.random.default_rng(abs(hash(name)) % (2**32) + 12).uniform(-1, 1, N)
    ud = dev(u)
    v = torch.full((N,), float("nan"), dtype=torch.float64, device="cuda")
    m.apply_advection_gll(ud, v, torch.empty_like(ud))
    assert_close(host(v), ogll.apply_advection_gll(spec, u), TOL_APPLY, name + " A_L")
    assert torch.equal(ud, dev(u)), "input modified"


@pytest.mark.parametrize("name", ["2d", "3d", "4d"])
def test_gll_config_full_parity(name):
    """BASELINE configs 2D/3D/4D at full size: the basis change, A_L and 10 RK steps on GLL coefficients."""
    import torch
    cfg = configs.CONFIGS[name]
    spec = cfg["spec"]
    u = inputs.full_vector(spec, cfg["recipe"], configs.seed_of(name))
    m = mesh(spec)
    ud = dev(u)
    v = torch.empty_like(ud)
    m.basis_change(ud, v, "gll_to_gauss")
    assert_close(host(v), ogll.basis_change(spec, u, "gll_to_gauss"), TOL_BASIS, name + " T")
    m.apply_advection_gll(ud, v, torch.empty_like(ud))
    assert_close(host(v), ogll.apply_advection_gll(spec, u), TOL_APPLY, name + " A_L")
    dt = configs.time_step(spec)
    bufs = [ud.clone(), torch.empty_like(ud), torch.empty_like(ud)]
    sol = m.rk_step_gll(bufs, 0, 0.0, dt, 10)
    assert_close(host(bufs[sol]), ogll.rk_steps_gll(spec, u, 0.0, dt, 10), TOL_RK10, name + " RK10 GLL")


def test_basis_change_6d_full_size_sampled():
    """Full-size 6D (4.1e9 DoFs) in the launch configuration the bench times: sampled cells against the oracle
    (the operation is cell-local), first and last cells included, and the round trip on the whole vector."""
    import torch
    cfg = configs.CONFIGS["6d"]
    spec = cfg["spec"]
    seed = configs.seed_of("6d")
    m = mesh(spec)
    N = m.owned_dofs
    nd = 4 ** 6
    u = torch.empty(N, dtype=torch.float64, device="cuda")
    m.fill_initial(u, cfg["recipe"], seed)
    v = torch.empty_like(u)
    m.basis_change(u, v, "gll_to_gauss")
    ncell = N // nd
    ids = np.unique(np.concatenate([[0, 1, ncell - 2, ncell - 1], np.random.default_rng(5).integers(0, ncell, 2048)]))
    one = dict(spec, cells=[1] * 6)     # the oracle's basis change only looks at d, n and the cell count
    own = inputs.cell_values(spec, cfg["recipe"], seed, ids)
    ref = ogll.basis_change(one, own.reshape(-1), "gll_to_gauss").reshape(len(ids), nd)
    got = host(v.view(-1, nd)[torch.from_numpy(ids).cuda()])
    assert_close(got, ref, TOL_BASIS, "6d T sampled")
    m.basis_change(v, v, "gauss_to_gll")
    d = (v - u).abs().max().item() / u.abs().max().item()
    assert d <= TOL_BASIS, f"6d round trip rel-max {d:.3e}"


def test_basis_change_rejects_bad_calls():
    import torch
    from paper_2002_08110_b200._binding import HDError
    spec = spec_of(1, 1, 2, [3, 2], [0.0, -1.0], [1.0, 1.0], [1.0, 0.5])
    m = mesh(spec)
    u = torch.zeros(2 * m.owned_dofs, dtype=torch.float64, device="cuda")
    a, b = u[:m.owned_dofs], u[2:m.owned_dofs + 2]
    with pytest.raises(HDError):
        m.basis_change(a, b, 0)          # partial overlap
    with pytest.raises(HDError):
        m.basis_change(a, a, 7)          # unknown kind
    with pytest.raises(HDError):
        m.apply_advection_gll(a, u[m.owned_dofs:], a)   # work aliases u


@pytest.mark.parametrize("P,xparts,vparts", [(2, None, None), (4, [2, 1], [1, 2])])
def test_basis_change_on_partitioned_meshes(P, xparts, vparts):
    """The basis change is cell-local: on the ranks of an x-slab and of a checkerboard x-v partition it equals the
    single-rank result bitwise, and the oracle to 1e-13 (hd.h: "any partition")."""
    import torch
    from paper_2002_08110_b200 import Mesh, configs
    from test_gpu_multirank import _join, _split, _vlasov
    spec = _vlasov(2, 2, 3, [4, 6, 2, 4], extra=0.1)
    u = np.random.default_rng(21).uniform(-1, 1, configs.dof_count(spec))
    one = Mesh(spec)
    ud = dev(u)
    ref = torch.empty_like(ud)
    one.basis_change(ud, ref, "gll_to_gauss")
    meshes = [Mesh(spec, rank=r, nranks=P, xparts=xparts, vparts=vparts) for r in range(P)]
    parts = _split(spec, u, meshes)
    outs = []
    for m, part in zip(meshes, parts):
        x = dev(part)
        m.basis_change(x, x, "gll_to_gauss")
        outs.append(host(x))
    got = _join(spec, outs, meshes)
    assert np.array_equal(got, host(ref))
    assert_close(got, ogll.basis_change(spec, u, "gll_to_gauss"), TOL_BASIS, "partitioned T")
