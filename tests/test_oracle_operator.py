"""Pins for the oracle's advection / mass operators (SURVEY 8(c) "What pins each part").

O2 (C++ literal ECL, oracle/hd_oracle.cpp) is checked against
  * a closed form derived by hand (tests/golden/adv1d_k1_two_cells.txt),
  * O1 dense over-integrated assembly and O3 Kronecker sum on tiny meshes,
  * invariants: constant state, conservation, exact upwind energy
    identity, k = 0 first-order upwind finite volumes, M^-1 M = I.
"""
import itertools

import numpy as np
import pytest

from conftest import load_golden
from oracle import capi, dense, kron


def spec_of(d_x, d_v, k, cells, lo, hi, a_const, a_lin=None, flux="upwind"):
    d = d_x + d_v
    if a_lin is None:
        a_lin = [[0.0] * d for _ in range(d)]
    return dict(d_x=d_x, d_v=d_v, k=k, cells=cells, lo=lo, hi=hi, a_const=a_const, a_lin=a_lin, flux=flux)


def tiny_spec(d, k, vlasov, flux="upwind"):
    """Tiny meshes with unequal cell sizes per dim; Vlasov-like fields keep v = 0 on a
    cell boundary so that sign(a.n) is constant per face (reading C11)."""
    if d == 2:
        d_x, d_v, cells = 1, 1, [3, 2]
    elif d == 3:
        d_x, d_v, cells = 2, 1, [2, 3, 2]
    else:
        d_x, d_v, cells = 2, 2, ([2, 2, 2, 2] if k < 3 else [2, 1, 2, 2])
    lo = [0.0, 0.2, -2.0, -1.5][:d]
    hi = [1.3, 0.9, 2.0, 1.5][:d]
    if not vlasov:
        return spec_of(d_x, d_v, k, cells, lo, hi, [1.0, -0.6, 0.45, -0.8][:d], flux=flux)
    # x-dims ride on the v coordinates; v-dims constant or x-dependent
    if d == 2:
        lo, hi = [0.0, -2.0], [1.3, 2.0]
        a_const = [0.0, 0.3]
        a_lin = [[0, 1.0], [0, 0]]
    elif d == 3:
        lo, hi = [0.0, 0.2, -2.0], [1.3, 0.9, 2.0]
        a_const = [0.0, 0.0, -0.25]
        a_lin = [[0, 0, 1.0], [0, 0, -0.5], [0, 0, 0]]
    else:
        lo, hi = [0.0, 0.2, -2.0, -1.5], [1.3, 0.9, 2.0, 1.5]
        a_const = [0.0, 0.0, 0.3, -0.2]
        a_lin = [[0, 0, 1.0, 0], [0, 0, 0, 1.0], [0.5, 0, 0, 0], [0, 0, 0, 0]]
    return spec_of(d_x, d_v, k, cells, lo, hi, a_const, a_lin, flux=flux)


def rel_max(a, b):
    return np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)


def test_worked_example_closed_form():
    rows = load_golden("adv1d_k1_two_cells.txt")
    expected = np.zeros((4, 4))
    for r, c, p, q in rows:
        expected[int(r), int(c)] = float(p) + float(q) * np.sqrt(3.0)
    spec = spec_of(1, 0, 1, [2], [0.0], [1.0], [1.0])
    N = 4
    got = np.column_stack([capi.apply_advection(spec, np.eye(N)[j], merged=True) for j in range(N)])
    assert np.max(np.abs(got - expected)) < 1e-13
    assert np.max(np.abs(got.sum(axis=1))) < 1e-13  # rows sum to 0 (constant state)


@pytest.mark.parametrize("d,k,vlasov,flux",
                         [(d, k, v, "upwind") for d in (2, 3, 4) for k in (1, 2, 3) for v in (False, True)]
                         + [(2, 2, True, "central"), (3, 1, False, "central"), (3, 2, True, "central")])
def test_tiers_agree(d, k, vlasov, flux):
    spec = tiny_spec(d, k, vlasov, flux)
    N = capi.dof_count(spec)
    rng = np.random.default_rng(100 * d + 10 * k + vlasov)
    u = rng.uniform(-1, 1, N)
    v2 = capi.apply_advection(spec, u)
    v1 = dense.apply_advection(spec, u)
    assert rel_max(v2, v1) < 1e-12, "O2 vs O1 weak form"
    m2 = capi.apply_advection(spec, u, merged=True)
    m1 = dense.apply_advection(spec, u, merged=True)
    m3 = kron.apply_merged(spec, u)
    assert rel_max(m2, m1) < 1e-12, "O2 vs O1 merged"
    assert rel_max(m2, m3) < 1e-12, "O2 vs O3 merged"


def test_pointwise_upwind_with_sign_change_inside_cells():
    # a_0 = v changes sign inside v-cells (3 cells on [-1,1]): the definition is the
    # pointwise Gauss-point upwind flux (reading C11); O2 and O3 both implement it.
    spec = spec_of(1, 1, 2, [4, 3], [0.0, -1.0], [1.0, 1.0], [0.0, 0.4], [[0, 1.0], [0, 0]])
    N = capi.dof_count(spec)
    u = np.random.default_rng(5).uniform(-1, 1, N)
    assert rel_max(capi.apply_advection(spec, u, merged=True), kron.apply_merged(spec, u)) < 1e-12


def test_dense_mass_is_diagonal_collocated():
    # P:246-249 / C2: collocation on Gauss points => M = diag(|J| prod w)
    spec = tiny_spec(3, 2, False)
    _, M = dense.assemble(spec)
    off = M - np.diag(np.diag(M))
    assert np.max(np.abs(off)) < 1e-15 * np.max(np.abs(M)) * 10
    ones = np.ones(M.shape[0])
    assert rel_max(capi.apply_mass(spec, ones), np.diag(M)) < 1e-14


@pytest.mark.parametrize("d,vlasov", [(2, False), (3, True), (4, True)])
def test_constant_state_and_conservation(d, vlasov):
    spec = tiny_spec(d, 2, vlasov)
    N = capi.dof_count(spec)
    v = capi.apply_advection(spec, np.ones(N))
    scale = capi.apply_advection(spec, np.random.default_rng(1).uniform(-1, 1, N))
    assert np.max(np.abs(v)) < 1e-13 * np.max(np.abs(scale))
    u = np.random.default_rng(2).uniform(-1, 1, N)
    Au = capi.apply_advection(spec, u)
    assert abs(Au.sum()) < 1e-13 * np.sum(np.abs(Au))  # 1^T A(u) = 0


def _traces(spec, u):
    """Independent evaluation of all face traces (numpy leggauss Lagrange values)."""
    d = spec["d_x"] + spec["d_v"]
    n = spec["k"] + 1
    cells = spec["cells"]
    x, w = np.polynomial.legendre.leggauss(n)
    x, w = 0.5 * (x + 1), 0.5 * w
    l0 = np.array([np.prod([(0 - x[k]) / (x[j] - x[k]) for k in range(n) if k != j]) for j in range(n)])
    l1 = np.array([np.prod([(1 - x[k]) / (x[j] - x[k]) for k in range(n) if k != j]) for j in range(n)])
    shape = [cells[i] for i in reversed(range(d))] + [n] * d
    U = u.reshape(shape)
    return U, x, w, l0, l1, shape


def test_central_flux_is_skew():
    # with F* = (a.n)(u- + u+)/2 and div a = 0 the face terms cancel the volume term's boundary part:
    # u^T A_c(u) = 0 for every u (energy conservation of the semi-discrete central scheme); a one-sided
    # trace, a dropped face term or a wrong sign would leave the -1/2 sum |a.n| (u- - u+)^2 jump term
    for vlasov in (False, True):
        spec = dict(tiny_spec(3, 2, vlasov), flux="central")
        N = capi.dof_count(spec)
        for seed in (4, 5):
            u = np.random.default_rng(seed).uniform(-1, 1, N)
            v = capi.apply_advection(spec, u)
            assert abs(u @ v) <= 1e-13 * np.linalg.norm(u) * np.linalg.norm(v), (vlasov, u @ v)


def test_upwind_energy_identity():
    # u^T A(u) = -1/2 sum_faces sum_q w_f |J_f| |a.n| (u- - u+)^2 (exact for div a = 0)
    for vlasov in (False, True):
        spec = tiny_spec(3, 2, vlasov)
        d = 3
        N = capi.dof_count(spec)
        u = np.random.default_rng(3).uniform(-1, 1, N)
        lhs = u @ capi.apply_advection(spec, u)
        U, x, w, l0, l1, shape = _traces(spec, u)
        cells = spec["cells"]
        lo = np.array(spec["lo"])
        h = (np.array(spec["hi"]) - lo) / np.array(cells)
        Jdet = np.prod(h)
        rhs = 0.0
        for i in range(d):
            ca, ma = d - 1 - i, 2 * d - 1 - i
            V = np.moveaxis(U, (ca, ma), (0, 1))  # [cells_i, n, rest]
            um = np.tensordot(l1, V, axes=([0], [1]))          # trace at x_i = 1 of every cell
            up = np.tensordot(l0, np.roll(V, -1, axis=0), axes=([0], [1]))  # right neighbour at x_i = 0
            # face weights and speed at the face points (a_i independent of z_i)
            rest_shape = [s for j, s in enumerate(shape) if j not in (ca, ma)]
            grids = np.meshgrid(*[np.arange(s) for s in rest_shape], indexing="ij")
            rest_axes = [j for j in range(2 * d) if j not in (ca, ma)]
            wf = np.ones(rest_shape)
            z = [None] * d
            for ax, gidx in zip(rest_axes, grids):
                if ax >= d:  # node axis of dim 2d-1-ax
                    dim = 2 * d - 1 - ax
                    wf = wf * w[gidx]
            for dim in range(d):
                if dim == i:
                    continue
                cax, nax = d - 1 - dim, 2 * d - 1 - dim
                cg = grids[rest_axes.index(cax)]
                ng = grids[rest_axes.index(nax)]
                z[dim] = lo[dim] + (cg + x[ng]) * h[dim]
            a = np.full(rest_shape, spec["a_const"][i])
            for j in range(d):
                if spec["a_lin"][i][j] != 0:
                    a = a + spec["a_lin"][i][j] * z[j]
            rhs += -0.5 * np.sum(wf[None] * (Jdet / h[i]) * np.abs(a)[None] * (um - up) ** 2)
        assert abs(lhs - rhs) < 1e-12 * abs(rhs), (vlasov, lhs, rhs)


def test_k0_is_first_order_upwind_finite_volume():
    # k = 0: (M^-1 A u)_j = -(a/h)(u_j - u_{j-1}) for a > 0
    spec = spec_of(1, 0, 0, [7], [0.0], [2.0], [1.5])
    u = np.random.default_rng(4).uniform(-1, 1, 7)
    got = capi.apply_advection(spec, u, merged=True)
    assert np.max(np.abs(got - (-(1.5 / (2.0 / 7)) * (u - np.roll(u, 1))))) < 1e-13
    # 2D, a = (-0.7, 0.4): sum of two 1D upwind differences (left-going in x)
    spec = spec_of(1, 1, 0, [5, 4], [0, 0], [1, 2], [-0.7, 0.4])
    U = np.random.default_rng(6).uniform(-1, 1, (4, 5))  # [c1, c0]
    got = capi.apply_advection(spec, U.reshape(-1), merged=True).reshape(4, 5)
    exp = (0.7 / 0.2) * (np.roll(U, -1, axis=1) - U) - (0.4 / 0.5) * (U - np.roll(U, 1, axis=0))
    assert np.max(np.abs(got - exp)) < 1e-13


def test_mass_round_trip_and_closed_form():
    spec = tiny_spec(4, 2, True)
    N = capi.dof_count(spec)
    u = np.random.default_rng(7).uniform(-1, 1, N)
    back = capi.apply_inv_mass(spec, capi.apply_mass(spec, u))
    assert np.max(np.abs(back - u)) < 4e-16 * np.max(np.abs(u)) * 4
    # closed form M_qq = prod_i h_i w_{q_i}, DoF q of cell 0 (C2)
    x, w = np.polynomial.legendre.leggauss(3)
    w = 0.5 * w
    h = (np.array(spec["hi"]) - np.array(spec["lo"])) / np.array(spec["cells"])
    m = capi.apply_mass(spec, np.ones(N))
    for q in itertools.product(range(3), repeat=4):
        idx = sum(q[i] * 3**i for i in range(4))
        assert abs(m[idx] - np.prod(h) * np.prod([w[qi] for qi in q])) < 1e-16


def test_numerical_flux_examples():
    for kind, um, up, an, exp in load_golden("numerical_flux_examples.txt"):
        assert capi.numerical_flux(float(um), float(up), float(an), kind) == pytest.approx(float(exp), abs=1e-15)


def test_dof_counts_paper_table():
    for k, d, dofs in load_golden("dofs_per_cell_table.txt"):
        k, d = int(k), int(d)
        spec = spec_of(d // 2 + d % 2, d // 2, k, [1] * d, [0.0] * d, [1.0] * d, [0.0] * d)
        assert capi.dof_count(spec) == int(dofs)
    # configs of BASELINE.json: N = |C| (k+1)^d
    from paper_2002_08110_b200.configs import CONFIGS
    expected = {"2d": 1024, "3d": 4_096_000, "4d": 16_777_216, "5d": 254_803_968, "6d": 4_096_000_000}
    for name, cfg in CONFIGS.items():
        assert capi.dof_count(cfg["spec"]) == expected[name]


def test_sampled_cells_equal_full_apply():
    spec = tiny_spec(3, 2, True)
    N = capi.dof_count(spec)
    u = np.random.default_rng(8).uniform(-1, 1, N)
    full = capi.apply_advection(spec, u).reshape(-1, 27)
    from paper_2002_08110_b200.inputs import neighbour_ids
    ids = np.array([0, 5, 11])
    nb = neighbour_ids(spec, ids)
    U = u.reshape(-1, 27)
    cells = np.concatenate([U[ids][:, None, :], U[nb]], axis=1)
    got = capi.apply_advection_cells(spec, ids, cells)
    assert np.array_equal(got, full[ids])


def test_invalid_specs_rejected():
    bad = spec_of(1, 1, 2, [0, 2], [0, 0], [1, 1], [1, 1])
    with pytest.raises(ValueError):
        capi.dof_count(bad)
    bad = spec_of(1, 1, 2, [2, 2], [0, 0], [1, 1], [1, 1], a_lin=[[1.0, 0], [0, 0]])
    with pytest.raises(ValueError):
        capi.dof_count(bad)
