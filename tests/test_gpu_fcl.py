"""GPU parity of the face-centric loop (FCL) comparison path, hd_apply_advection_fcl (
P:579-600), against the CPU oracle (which evaluates every face from both sides, Alg. 2) and
against the element-centric product path. Same bar as the product operator: relative L2 and max error
<= 1e-12 per application (reading C17)."""
import numpy as np
import pytest

from oracle import capi as oracle
from paper_2002_08110_b200 import configs, inputs

from test_gpu_parity import (CENTRAL, DEGENERATE, SMALL, TOL_APPLY, _sampled_cells, assert_close, dev, host,
                             mesh, spec_of)

pytestmark = pytest.mark.gpu

CASES = SMALL + CENTRAL + [(n, s) for n, s in DEGENERATE if s["k"] + 1 >= 2]


@pytest.mark.parametrize("name,spec", CASES, ids=[s[0] for s in CASES])
def test_fcl_small_meshes(name, spec):
    """Every built (d, n), constant and Vlasov-like fields, upwind and central fluxes, fields whose sign
    changes inside cells (central), self-neighbours (one cell along a dim) and zero speeds."""
    import torch
    m = mesh(spec)
    N = m.owned_dofs
    u = np.random.default_rng(abs(hash(name)) % (2**32) + 7).uniform(-1, 1, N)
    ud = dev(u)
    vf = torch.full((N,), float("nan"), dtype=torch.float64, device="cuda")  # every entry must be written
    m.apply_advection_fcl(ud, vf)
    ref = oracle.apply_advection(spec, u)
    assert_close(host(vf), ref, TOL_APPLY, name + " FCL")
    ve = torch.empty_like(ud)
    m.apply_advection(ud, ve)
    assert_close(host(vf), host(ve), TOL_APPLY, name + " FCL vs ECL")
    # repeated call reuses the face buffers and gives the same bits
    vf2 = torch.empty_like(ud)
    m.apply_advection_fcl(ud, vf2)
    assert torch.equal(vf, vf2)


@pytest.mark.parametrize("name", ["2d", "3d", "4d"])
def test_fcl_config_full_parity(name):
    """The BASELINE configs 2D/3D/4D at full size, whole vector against the oracle."""
    import torch
    cfg = configs.CONFIGS[name]
    spec = cfg["spec"]
    u = inputs.full_vector(spec, cfg["recipe"], configs.seed_of(name))
    m = mesh(spec)
    ud = dev(u)
    vd = torch.empty_like(ud)
    m.apply_advection_fcl(ud, vd)
    assert_close(host(vd), oracle.apply_advection(spec, u), TOL_APPLY, name + " FCL")


def test_fcl_config_5d_sampled_parity():
    """Full-size 5D (255M DoFs; the FCL face buffers need 15 n^4 doubles per cell): sampled cells against
    the oracle cell by cell, and the whole vector against the (full-size parity-tested) ECL product path."""
    import torch
    cfg = configs.CONFIGS["5d"]
    spec = cfg["spec"]
    seed = configs.seed_of("5d")
    m = mesh(spec)
    N = m.owned_dofs
    u = torch.empty(N, dtype=torch.float64, device="cuda")
    m.fill_initial(u, cfg["recipe"], seed)
    vf = torch.empty_like(u)
    m.apply_advection_fcl(u, vf)
    ve = torch.empty_like(u)
    m.apply_advection(u, ve)
    d = (vf - ve).abs().max().item() / ve.abs().max().item()
    l2 = (torch.linalg.vector_norm(vf - ve) / torch.linalg.vector_norm(ve)).item()
    assert d <= TOL_APPLY and l2 <= TOL_APPLY, f"5d FCL vs ECL rel-max {d:.3e} rel-L2 {l2:.3e}"
    del ve
    nd = 4 ** 5
    ids = _sampled_cells(spec, 1024, np.random.default_rng(77))
    got = host(vf.view(-1, nd)[torch.from_numpy(ids).cuda()])
    own = inputs.cell_values(spec, cfg["recipe"], seed, ids)
    nb = inputs.neighbour_ids(spec, ids)
    nbv = inputs.cell_values(spec, cfg["recipe"], seed, nb.reshape(-1)).reshape(len(ids), -1, nd)
    ref = oracle.apply_advection_cells(spec, ids, np.concatenate([own[:, None, :], nbv], axis=1))
    assert_close(got, ref, TOL_APPLY, "5d sampled FCL")


def test_fcl_rejects_bad_calls():
    import torch
    from paper_2002_08110_b200._binding import HDError
    spec = spec_of(1, 1, 2, [3, 2], [0.0, -1.0], [1.0, 1.0], [1.0, 0.5])
    m = mesh(spec)
    u = torch.zeros(m.owned_dofs, dtype=torch.float64, device="cuda")
    with pytest.raises((HDError, ValueError)):
        m.apply_advection_fcl(u, u)  # aliasing
    with pytest.raises(ValueError):
        m.apply_advection_fcl(u, torch.zeros(m.owned_dofs - 1, dtype=torch.float64, device="cuda"))
