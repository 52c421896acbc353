"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Bar (BASELINE.json north_star, reading C17): relative L2 and relative max
error <= 1e-12 per operator application and <= 1e-10 after 10 RK steps. Inputs are the seeded
synthetic recipes of paper_2002_08110_b200/inputs.py; the oracle always receives them from numpy,
never from the GPU.
"""
import numpy as np
import pytest

from oracle import capi as oracle
from paper_2002_08110_b200 import configs, inputs

pytestmark = pytest.mark.gpu

TOL_APPLY = 1e-12
TOL_RK10 = 1e-10


def _torch():
    import torch
    return torch


def dev(x):
    torch = _torch()
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).cuda()


def host(t):
    _torch().cuda.synchronize()
    return t.cpu().numpy()


def errs(got, ref):
    d = got - ref
    l2 = np.linalg.norm(d) / max(np.linalg.norm(ref), 1e-300)
    mx = np.max(np.abs(d)) / max(np.max(np.abs(ref)), 1e-300)
    return l2, mx


def assert_close(got, ref, tol, what=""):
    l2, mx = errs(got, ref)
    assert l2 <= tol and mx <= tol, f"{what}: rel-L2 {l2:.3e} rel-max {mx:.3e} (tol {tol:.0e})"


def mesh(spec):
    from paper_2002_08110_b200 import Mesh
    return Mesh(spec)


def spec_of(d_x, d_v, k, cells, lo, hi, a_const, a_lin=None):
    d = d_x + d_v
    if a_lin is None:
        a_lin = [[0.0] * d for _ in range(d)]
    return dict(d_x=d_x, d_v=d_v, k=k, cells=list(cells), lo=list(lo), hi=list(hi), a_const=list(a_const),
                a_lin=[list(r) for r in a_lin], flux="upwind")


def small_specs():
    """Tiny meshes spanning every built (d, n), both field kinds, negative speeds, unequal h and
    ragged last batches."""
    out = []
    for d in range(2, 7):
        d_x = (d + 1) // 2
        d_v = d - d_x
        for k in range(1, 6):
            n = k + 1
            if n ** d > 4096 or n ** (d - 2) > 256:
                continue
            cells = [3, 2, 2, 3, 2, 2][:d] if n ** d <= 1296 else [2] * d
            lo = [0.0, 0.1, -0.5, -2.0, -1.0, -1.5][:d]
            hi = [1.0, 0.8, 0.7, 2.0, 1.0, 1.5][:d]
            a_const = [1.0, -0.7, 0.45, -0.3, 0.25, -0.6][:d]
            out.append((f"d{d}k{k}const", spec_of(d_x, d_v, k, cells, lo, hi, a_const)))
            # Vlasov-like: x dims ride on v coordinates (v boxes symmetric, even cell counts)
            lin = [[0.0] * d for _ in range(d)]
            vcells = list(cells)
            vlo, vhi = list(lo), list(hi)
            for i in range(min(d_x, d_v)):
                lin[i][d_x + i] = 1.0
            for j in range(d_x, d):
                vcells[j] = 2
                vlo[j], vhi[j] = -1.5 - 0.2 * j, 1.5 + 0.2 * j
            ac = [0.0] * d_x + [0.3, -0.2, 0.1][:d_v]
            if d_x > d_v:
                ac[d_x - 1] = 0.5
            if d >= 4:
                lin[d_x][0] = 0.2  # a v-component depending on x (keeps its sign on the box)
            out.append((f"d{d}k{k}vlasov", spec_of(d_x, d_v, k, vcells, vlo, vhi, ac, lin)))
    return out


SMALL = small_specs()


@pytest.mark.parametrize("name,spec", SMALL, ids=[s[0] for s in SMALL])
def test_small_mesh_operators(name, spec):
    torch = _torch()
    m = mesh(spec)
    N = m.owned_dofs
    rng = np.random.default_rng(abs(hash(name)) % (2**32))
    u = rng.uniform(-1, 1, N)
    ud, vd = dev(u), torch.empty(N, dtype=torch.float64, device="cuda")
    m.apply_advection(ud, vd)
    assert_close(host(vd), oracle.apply_advection(spec, u), TOL_APPLY, name + " A")
    # merged operator through the C ABI: M^-1 (A u)
    m.apply_inv_mass(vd)
    assert_close(host(vd), oracle.apply_advection(spec, u, merged=True), TOL_APPLY, name + " M^-1 A")
    w = dev(u)
    m.apply_inv_mass(w)
    assert_close(host(w), oracle.apply_inv_mass(spec, u), 1e-14, name + " M^-1")
    m.apply_mass(w)
    assert_close(host(w), u, 1e-14, name + " M M^-1")


@pytest.mark.parametrize("name,spec", SMALL[::3], ids=[s[0] for s in SMALL[::3]])
def test_small_mesh_rk10(name, spec):
    torch = _torch()
    m = mesh(spec)
    N = m.owned_dofs
    u = np.random.default_rng(7).uniform(-1, 1, N)
    dt = configs.time_step(spec, 0.1)
    bufs = [dev(u), torch.empty(N, dtype=torch.float64, device="cuda"),
            torch.empty(N, dtype=torch.float64, device="cuda")]
    sol = m.rk_step(bufs, 0, 0.0, dt, nsteps=10)
    ref = oracle.rk_steps(spec, u, 0.0, dt, 10)
    assert_close(host(bufs[sol]), ref, TOL_RK10, name + " rk10")


def central_specs():
    """Central-flux cases (reading C3): constant and Vlasov fields over d = 2..6, plus a field whose sign
    changes inside cells (allowed with the central flux, which never selects a side)."""
    out = []
    for name, spec in SMALL:
        d, k = len(spec["cells"]), spec["k"]
        if (d, k) in ((2, 3), (3, 2), (4, 1), (4, 2), (5, 1), (6, 1)):
            out.append((name + "central", dict(spec, flux="central")))
    out.append(("d2k3signchange", dict(spec_of(1, 1, 3, [4, 3], [0.0, -1.0], [1.0, 1.0], [0.0, 0.3],
                                               [[0, 1.0], [0, 0]]), flux="central")))
    out.append(("d4k2signchange", dict(spec_of(2, 2, 2, [3, 2, 3, 3], [0.0, 0.0, -1.0, -1.2], [1.0, 2.0, 1.0, 1.2],
                                               [0.0, 0.0, 0.25, -0.1],
                                               [[0, 0, 1, 0], [0, 0, 0, 1], [0.4, 0, 0, 0], [0, 0.3, 0, 0]]),
                                       flux="central")))
    return out


CENTRAL = central_specs()


@pytest.mark.parametrize("name,spec", CENTRAL, ids=[s[0] for s in CENTRAL])
def test_central_flux_operators_and_rk10(name, spec):
    """NEXT-3: v <- A_c(u) and 10 LSRK steps with the central flux against the oracle (which evaluates
    F* = (a.n)(u- + u+)/2 directly per face)."""
    torch = _torch()
    m = mesh(spec)
    N = m.owned_dofs
    rng = np.random.default_rng(abs(hash(name)) % (2**32))
    u = rng.uniform(-1, 1, N)
    ud, vd = dev(u), torch.empty(N, dtype=torch.float64, device="cuda")
    vd.fill_(float("nan"))  # the second half-launch accumulates into the first's output
    m.apply_advection(ud, vd)
    ref = oracle.apply_advection(spec, u)
    assert_close(host(vd), ref, TOL_APPLY, name + " A_c")
    ref_up = oracle.apply_advection(dict(spec, flux="upwind"), u)
    assert np.max(np.abs(ref_up - ref)) > 1e-3 * np.max(np.abs(ref))  # the flux matters on these inputs
    dt = configs.time_step(spec, 0.1)
    bufs = [dev(u), torch.empty(N, dtype=torch.float64, device="cuda"),
            torch.empty(N, dtype=torch.float64, device="cuda")]
    sol = m.rk_step(bufs, 0, 0.0, dt, nsteps=10)
    assert_close(host(bufs[sol]), oracle.rk_steps(spec, u, 0.0, dt, 10), TOL_RK10, name + " rk10")
    # the central-flux operator is skew (u^T A_c u = 0 for a divergence-free field), so the semi-discrete
    # system conserves u^T M u and ten LSRK steps at CFL 0.1 change it only by the method's dissipation (~1e-9)
    assert abs(float(np.dot(u, host(vd)))) <= 1e-12 * float(np.linalg.norm(ref)) * np.sqrt(N)
    w = dev(u)
    m.apply_mass(w)
    e0 = float(np.dot(u, host(w)))
    w = bufs[sol].clone()
    m.apply_mass(w)
    e1 = float(np.dot(host(bufs[sol]), host(w)))
    assert abs(e1 - e0) <= 1e-7 * e0, (e0, e1)


def test_constant_state_and_conservation_on_gpu():
    torch = _torch()
    spec = configs.CONFIGS["5d"]["spec"]
    small = dict(spec, cells=[4, 4, 4, 4, 4])
    m = mesh(small)
    N = m.owned_dofs
    ones = torch.ones(N, dtype=torch.float64, device="cuda")
    v = torch.empty_like(ones)
    m.apply_advection(ones, v)
    u = dev(np.random.default_rng(3).uniform(-1, 1, N))
    w = torch.empty_like(u)
    m.apply_advection(u, w)
    scale = float(w.abs().max())
    assert float(v.abs().max()) < 1e-13 * scale
    assert abs(float(w.sum())) < 1e-13 * float(w.abs().sum())


@pytest.mark.parametrize("name", ["2d", "3d", "4d"])
def test_config_full_parity(name):
    torch = _torch()
    cfg = configs.CONFIGS[name]
    spec = cfg["spec"]
    u = inputs.full_vector(spec, cfg["recipe"], configs.seed_of(name))
    m = mesh(spec)
    N = m.owned_dofs
    assert N == u.size
    ud = dev(u)
    vd = torch.empty_like(ud)
    m.apply_advection(ud, vd)
    assert_close(host(vd), oracle.apply_advection(spec, u), TOL_APPLY, name + " A")
    w = dev(u)
    m.apply_inv_mass(w)
    assert_close(host(w), oracle.apply_inv_mass(spec, u), 1e-14, name + " M^-1")
    # 10 RK steps (north star: <= 1e-10)
    dt = configs.time_step(spec, cfg["cfl"])
    bufs = [dev(u), torch.empty_like(ud), torch.empty_like(ud)]
    sol = m.rk_step(bufs, 0, 0.0, dt, nsteps=10)
    ref = oracle.rk_steps(spec, u, 0.0, dt, 10)
    assert_close(host(bufs[sol]), ref, TOL_RK10, name + " rk10")


def test_config_5d_full_apply_and_rk10():
    """Full-size 5D (255M DoFs, the bench's 5D launch configuration: pencil units of CT = 4 cells): one
    apply_advection and 10 LSRK steps against the oracle on the whole vector (north star: <= 1e-12 per
    application, <= 1e-10 after 10 steps; the oracle RK10 takes a few minutes on the host cores)."""
    torch = _torch()
    cfg = configs.CONFIGS["5d"]
    spec = cfg["spec"]
    seed = configs.seed_of("5d")
    u = inputs.full_vector(spec, cfg["recipe"], seed)
    m = mesh(spec)
    ud = dev(u)
    vd = torch.empty_like(ud)
    m.apply_advection(ud, vd)
    got = host(vd)
    del vd
    assert_close(got, oracle.apply_advection(spec, u), TOL_APPLY, "5d A")
    # GPU-side generator equals the numpy recipe
    g = torch.empty_like(ud)
    m.fill_initial(g, cfg["recipe"], seed)
    assert_close(host(g), u, 1e-14, "5d fill")
    del g, got
    dt = configs.time_step(spec, cfg["cfl"])
    bufs = [ud, torch.empty_like(ud), torch.empty_like(ud)]
    sol = m.rk_step(bufs, 0, 0.0, dt, nsteps=10)
    got = host(bufs[sol])
    del bufs, ud
    assert_close(got, oracle.rk_steps(spec, u, 0.0, dt, 10), TOL_RK10, "5d rk10")


def _sampled_cells(spec, count, rng):
    d = spec["d_x"] + spec["d_v"]
    L = np.array(spec["cells"])
    ncell = int(np.prod(L))
    ids = set(rng.integers(0, ncell, count).tolist())
    # every kind of periodic boundary cell: corners of the index box plus faces
    strides = np.concatenate([[1], np.cumprod(L)[:-1]])
    for corner in range(1 << d):
        c = np.array([(L[i] - 1) if (corner >> i) & 1 else 0 for i in range(d)])
        ids.add(int(c @ strides))
    for i in range(d):
        for edge in (0, L[i] - 1):
            c = rng.integers(0, L)
            c[i] = edge
            ids.add(int(c @ strides))
    return np.array(sorted(ids), dtype=np.int64)


def test_config_6d_sampled_parity():
    """Full-size 6D (4.1e9 DoFs, 32.8 GB per vector, 64-bit indexing) in the launch configuration the
    bench times; >= 4096 random cells plus boundary cells are recomputed by the oracle cell by cell."""
    torch = _torch()
    cfg = configs.CONFIGS["6d"]
    spec = cfg["spec"]
    seed = configs.seed_of("6d")
    m = mesh(spec)
    N = m.owned_dofs
    assert N == 4_096_000_000
    u = torch.empty(N, dtype=torch.float64, device="cuda")
    m.fill_initial(u, cfg["recipe"], seed)
    v = torch.empty_like(u)
    m.apply_advection(u, v)
    rng = np.random.default_rng(2024)
    ids = _sampled_cells(spec, 4096, rng)
    nd = 4 ** 6
    idx = torch.from_numpy(ids).cuda()
    got = host(v.view(-1, nd)[idx])
    gu = host(u.view(-1, nd)[idx])
    del v
    own = inputs.cell_values(spec, cfg["recipe"], seed, ids)
    assert_close(gu, own, 1e-14, "6d fill vs numpy")
    nb = inputs.neighbour_ids(spec, ids)
    nbv = inputs.cell_values(spec, cfg["recipe"], seed, nb.reshape(-1)).reshape(len(ids), -1, nd)
    cells = np.concatenate([own[:, None, :], nbv], axis=1)
    ref = oracle.apply_advection_cells(spec, ids, cells)
    assert_close(got, ref, TOL_APPLY, "6d sampled A")
    # in-place inverse mass on the full vector, sampled
    m.apply_inv_mass(u)
    # the mass depends only on h and the cell-local index: compute it on a one-cell mesh with the
    # same h (lo/hi rescaled), then compare the sampled cells
    h = (np.array(spec["hi"]) - np.array(spec["lo"])) / np.array(spec["cells"])
    one = dict(spec, cells=[1] * 6, lo=[0.0] * 6, hi=list(h), a_lin=[[0.0] * 6 for _ in range(6)],
               a_const=[0.0] * 6)
    ref_im = np.stack([oracle.apply_inv_mass(one, own[i]) for i in range(len(ids))])
    assert_close(host(u.view(-1, nd)[idx]), ref_im, 1e-14, "6d sampled M^-1")


def _gather_cells(vec, nd, ids):
    torch = _torch()
    return host(vec.view(-1, nd)[torch.from_numpy(np.ascontiguousarray(ids, dtype=np.int64)).cuda()])


def test_config_6d_rk_stages_sampled_parity():
    """Full-size 6D RK stages in the bench's launch configuration (cell_kernel<6,4,RK>, 10^6 cells, pencil
    units, skew 2, published traces, direct-read fallbacks): every one of the 5 stages of a step is run
    through hd_rk_stage and, on >= 1024 random cells plus boundary cells, compared with the oracle's merged
    operator of the sampled cells (given U and its neighbours) followed by the 2N update."""
    torch = _torch()
    cfg = configs.CONFIGS["6d"]
    spec = cfg["spec"]
    m = mesh(spec)
    N = m.owned_dofs
    nd = 4 ** 6
    dt = configs.time_step(spec, cfg["cfl"])
    A, B, _ = oracle.rk_coefficients()
    bufs = [torch.empty(N, dtype=torch.float64, device="cuda") for _ in range(3)]
    m.fill_initial(bufs[0], cfg["recipe"], configs.seed_of("6d"))
    iu, idu, iw = 0, 1, 2
    rng = np.random.default_rng(606)
    for s in range(5):
        ids = _sampled_cells(spec, 1024, rng)
        nb = inputs.neighbour_ids(spec, ids)
        U = bufs[iu]
        own = _gather_cells(U, nd, ids)
        nbv = _gather_cells(U, nd, nb.reshape(-1)).reshape(len(ids), -1, nd)
        du_in = _gather_cells(bufs[idu], nd, ids) if s > 0 else np.zeros_like(own)
        m.rk_stage(U, bufs[idu], bufs[iw], s, dt)
        got_du = _gather_cells(bufs[idu], nd, ids)
        got_u = _gather_cells(bufs[iw], nd, ids)
        r = oracle.apply_advection_cells(spec, ids, np.concatenate([own[:, None, :], nbv], axis=1), merged=True)
        ref_du = A[s] * du_in + dt * r
        ref_u = own + B[s] * ref_du
        assert_close(got_du, ref_du, TOL_APPLY, f"6d stage {s} dU")
        assert_close(got_u, ref_u, TOL_APPLY, f"6d stage {s} U")
        iu, iw = iw, iu


def test_6d_full_rk_step_conserves_mass():
    torch = _torch()
    cfg = configs.CONFIGS["6d"]
    spec = cfg["spec"]
    m = mesh(spec)
    N = m.owned_dofs
    bufs = [torch.empty(N, dtype=torch.float64, device="cuda") for _ in range(3)]
    m.fill_initial(bufs[0], cfg["recipe"], configs.seed_of("6d"))
    w = bufs[0].clone()
    m.apply_mass(w)
    mass0 = float(w.sum())
    del w
    dt = configs.time_step(spec, cfg["cfl"])
    sol = m.rk_step(bufs, 0, 0.0, dt, nsteps=1)
    assert sol == 2
    out = bufs[sol]
    assert bool(torch.isfinite(out).all())
    w = out.clone()
    m.apply_mass(w)
    assert abs(float(w.sum()) - mass0) < 1e-12 * abs(mass0)


def test_fill_matches_numpy_small_configs():
    torch = _torch()
    for name in ("2d", "3d", "4d"):
        cfg = configs.CONFIGS[name]
        spec = cfg["spec"]
        m = mesh(spec)
        g = torch.empty(m.owned_dofs, dtype=torch.float64, device="cuda")
        m.fill_initial(g, cfg["recipe"], configs.seed_of(name))
        assert_close(host(g), inputs.full_vector(spec, cfg["recipe"], configs.seed_of(name)), 1e-14, name)


def test_rk_host_variant_and_rotation():
    torch = _torch()
    spec = configs.CONFIGS["2d"]["spec"]
    m = mesh(spec)
    N = m.owned_dofs
    u = inputs.full_vector(spec, "gauss2d", 7)
    dt = configs.time_step(spec, 0.1)
    bufs = [dev(u), torch.empty(N, dtype=torch.float64, device="cuda"),
            torch.empty(N, dtype=torch.float64, device="cuda")]
    sol = m.rk_step(bufs, 0, 0.0, dt, nsteps=3)
    assert sol == 2  # 15 stages, odd: solution ends in the rotation partner
    hu = torch.from_numpy(u.copy()).pin_memory()
    out = torch.empty(N, dtype=torch.float64).pin_memory()
    dbufs = [torch.empty(N, dtype=torch.float64, device="cuda") for _ in range(3)]
    m.rk_step_host(hu, out, dbufs, 0.0, dt, nsteps=3)
    assert np.array_equal(out.numpy(), host(bufs[sol]))


def test_aliasing_is_rejected():
    torch = _torch()
    from paper_2002_08110_b200 import HDError
    m = mesh(configs.CONFIGS["2d"]["spec"])
    u = torch.zeros(m.owned_dofs, dtype=torch.float64, device="cuda")
    with pytest.raises(HDError):
        m.apply_advection(u, u)
    with pytest.raises(HDError):
        m.rk_step([u, u, torch.zeros_like(u)], 0, 0.0, 1e-3)


DEGENERATE = [
    # a single cell (every neighbour is the cell itself, periodic)
    ("one-cell-4d", spec_of(2, 2, 3, [1, 1, 1, 1], [0.0, 0.0, -1.0, -1.0], [1.0, 1.0, 1.0, 1.0],
                            [0.7, -0.4, 0.3, -0.2])),
    # length-1 dims mixed with longer ones, pencil mode (6D) and groups across pencils (5D)
    ("thin-6d", spec_of(3, 3, 3, [3, 1, 2, 1, 2, 2], [0.0] * 6, [1.0] * 6, [0.9, -0.5, 0.4, -0.3, 0.2, -0.6])),
    ("thin-5d", spec_of(3, 2, 3, [5, 4, 1, 2, 2], [0.0] * 5, [1.0] * 5, [-0.9, 0.5, 0.4, -0.3, 0.2])),
    # speeds exactly zero in some dims (no flux along them)
    ("zero-speed-4d", spec_of(2, 2, 3, [3, 2, 2, 3], [0.0] * 4, [1.0] * 4, [0.0, 0.8, 0.0, -0.5])),
    # k = 1 and k = 5 at the sizes the kernels allow
    ("k1-6d", spec_of(3, 3, 1, [3, 2, 2, 3, 2, 2], [0.0] * 6, [1.0] * 6, [0.5, -0.4, 0.3, -0.2, 0.6, -0.1])),
    ("k5-4d", spec_of(2, 2, 5, [2, 3, 2, 2], [0.0] * 4, [1.0] * 4, [0.5, -0.4, 0.3, -0.2])),
    # pencils longer than one group: a_0 = v_0 = z_1 (chunk mode: part of a pencil per group, the
    # pencils of a group would sweep dim 0 in opposite directions) ...
    ("long-x-2d-vlasov", spec_of(1, 1, 1, [520, 4], [0.0, -1.5], [1.0, 1.5], [0.0, 0.3],
                                 [[0.0, 1.0], [0.0, 0.0]])),
    ("long-x-3d-vlasov", spec_of(1, 2, 3, [70, 2, 2], [0.0, -1.0, -1.0], [1.0, 1.0, 1.0], [0.0, 0.3, -0.2],
                                 [[0.0, 1.0, 0.0], [0.0] * 3, [0.0] * 3])),
    ("long-x-4d-vlasov", spec_of(1, 3, 3, [20, 2, 2, 2], [0.0, -1.0, -1.0, -1.0], [1.0] * 4,
                                 [0.0, 0.3, -0.2, 0.1], [[0.0, 1.0, 0.0, 0.0]] + [[0.0] * 4] * 3)),
    # ... and a_0 independent of z_1 (pencil mode in 2D/3D, dim-0 carry, following dims)
    ("long-x-2d-const", spec_of(1, 1, 1, [300, 3], [0.0, 0.0], [1.0, 1.0], [-0.8, 0.6])),
    ("long-x-3d-pencil", spec_of(2, 1, 3, [70, 4, 2], [0.0, 0.0, -1.0], [1.0, 1.0, 1.0], [0.0, 0.4, 0.3],
                                 [[0.0, 0.0, 1.0], [0.0] * 3, [0.0] * 3])),
]


@pytest.mark.parametrize("name,spec", DEGENERATE, ids=[s[0] for s in DEGENERATE])
def test_degenerate_meshes(name, spec):
    """Edge cases of the method: self-neighbours (one cell along a dim), zero speeds, extreme degrees."""
    torch = _torch()
    m = mesh(spec)
    N = m.owned_dofs
    u = np.random.default_rng(5).uniform(-1, 1, N)
    ud, vd = dev(u), torch.empty(N, dtype=torch.float64, device="cuda")
    m.apply_advection(ud, vd)
    assert_close(host(vd), oracle.apply_advection(spec, u), TOL_APPLY, name + " A")
    dt = 1e-3
    bufs = [dev(u), torch.empty_like(ud), torch.empty_like(ud)]
    sol = m.rk_step(bufs, 0, 0.0, dt, nsteps=10)
    assert_close(host(bufs[sol]), oracle.rk_steps(spec, u, 0.0, dt, 10), TOL_RK10, name + " rk10")


def test_repeated_launches_reuse_flags():
    """Many launches on one mesh (progress flags carry the launch epoch): results stay exact."""
    torch = _torch()
    cfg = configs.CONFIGS["5d"]
    spec = dict(cfg["spec"], cells=[6, 6, 6, 4, 4])
    m = mesh(spec)
    u = inputs.full_vector(spec, cfg["recipe"], configs.seed_of("5d"))
    ud = dev(u)
    ref = oracle.apply_advection(spec, u)
    v = torch.empty_like(ud)
    for _ in range(7):
        m.apply_advection(ud, v)
    assert_close(host(v), ref, TOL_APPLY, "repeated A")
