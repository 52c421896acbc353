"""GPU: the multi-rank path (x-space and checkerboard x-v partitions + upwind-trace halo with the v-chunk
pipeline) against one rank and
against the oracle, with all ranks' meshes on one device and the in-process loopback transport (the
same buffers NCCL would fill; one GPU is all this pool gives, and ranks must not spin on each other).

C18: the per-cell arithmetic does not depend on the partition, so P > 1 must equal P = 1 BITWISE;
the oracle bar is the usual 1e-12 (application) / 1e-10 (10 RK steps).
"""
import numpy as np
import pytest

from oracle import capi as oracle
from paper_2002_08110_b200 import Mesh, apply_advection_group, configs, inputs, rk_step_group

pytestmark = pytest.mark.gpu


def _spec(d_x, d_v, k, cells, lo, hi, a_const, a_lin=None):
    d = d_x + d_v
    if a_lin is None:
        a_lin = [[0.0] * d for _ in range(d)]
    return dict(d_x=d_x, d_v=d_v, k=k, cells=list(cells), lo=list(lo), hi=list(hi), a_const=list(a_const),
                a_lin=[list(r) for r in a_lin], flux="upwind")


def _vlasov(d_x, d_v, k, cells, vmax=2.0, extra=0.0):
    d = d_x + d_v
    lin = [[0.0] * d for _ in range(d)]
    for i in range(min(d_x, d_v)):
        lin[i][d_x + i] = 1.0
    if extra:
        lin[d_x][0] = extra  # a v-speed that depends on x (keeps its sign on the box)
    ac = [0.0] * d_x + [0.3, -0.2, 0.1][:d_v]
    if d_x > d_v:
        ac[d_x - 1] = 0.5
    return _spec(d_x, d_v, k, cells, [0.0] * d_x + [-vmax] * d_v, [1.0] * d_x + [vmax] * d_v, ac, lin)


# (name, spec, P, xparts, vparts)
CASES = [
    ("3d-const-P2", _spec(2, 1, 4, [4, 6, 3], [0] * 3, [1] * 3, [1.0, -0.7, 0.3]), 2, None, None),
    ("4d-vlasov-P2", _vlasov(2, 2, 3, [4, 6, 2, 4], extra=0.1), 2, None, None),
    ("4d-vlasov-P4", _vlasov(2, 2, 3, [4, 6, 2, 4], extra=0.1), 4, None, None),
    ("5d-vlasov-P2", _vlasov(3, 2, 3, [6, 6, 6, 4, 4]), 2, None, None),
    ("5d-vlasov-P8", _vlasov(3, 2, 3, [6, 6, 6, 4, 4]), 8, None, None),
    ("5d-vlasov-P3-x0", _vlasov(3, 2, 3, [6, 6, 6, 4, 4]), 3, [3, 1, 1], None),
    ("6d-vlasov-P8", _vlasov(3, 3, 3, [4, 4, 4, 2, 2, 2]), 8, None, None),
    # long pencils with a_0 = v_0 = z_1: chunk mode (parts of a pencil per group) with the dim-0 halo
    ("2d-vlasov-chunk-P2", _vlasov(1, 1, 1, [1040, 4]), 2, None, None),
    ("3d-vlasov-chunk-P2", _vlasov(1, 2, 3, [140, 2, 2]), 2, None, None),
    # checkerboard x-v partitions (NEXT-4): v dims split too, halo along v dims
    ("4d-vlasov-P4-xv", _vlasov(2, 2, 3, [4, 6, 2, 4], extra=0.1), 4, [2, 1], [1, 2]),
    ("5d-vlasov-P4-v", _vlasov(3, 2, 3, [6, 6, 6, 4, 4]), 4, [1, 1, 1], [2, 2]),
    ("5d-vlasov-P4-xv", _vlasov(3, 2, 3, [6, 6, 6, 4, 4]), 4, [1, 1, 2], [2, 1]),
    ("6d-vlasov-P8-xv", _vlasov(3, 3, 3, [4, 4, 4, 2, 2, 2]), 8, [1, 2, 1], [2, 1, 2]),
]


def _cells_view(spec, u):
    d = spec["d_x"] + spec["d_v"]
    nd = (spec["k"] + 1) ** d
    return u.reshape(list(spec["cells"][::-1]) + [nd])  # [c_{d-1}, ..., c_0, dof]


def _box(spec, m):
    d = spec["d_x"] + spec["d_v"]
    return tuple(slice(m.box_off[i], m.box_off[i] + m.box_len[i]) for i in reversed(range(d)))


def _split(spec, u, meshes):
    cv = _cells_view(spec, u)
    return [np.ascontiguousarray(cv[_box(spec, m)]).reshape(-1) for m in meshes]


def _join(spec, parts, meshes):
    out = np.full(_cells_view(spec, np.zeros(sum(p.size for p in parts))).shape, np.nan)
    for p, m in zip(parts, meshes):
        out[_box(spec, m)] = p.reshape(out[_box(spec, m)].shape)
    return out.reshape(-1)


@pytest.mark.parametrize("name,spec,P,xparts,vparts", CASES, ids=[c[0] for c in CASES])
def test_partitioned_equals_single_rank_bitwise(name, spec, P, xparts, vparts):
    import torch
    u = np.random.default_rng(11).uniform(-1, 1, configs.dof_count(spec))
    one = Mesh(spec)
    ud = torch.from_numpy(u).cuda()
    vd = torch.empty_like(ud)
    one.apply_advection(ud, vd)
    ref_a = vd.cpu().numpy()
    dt = configs.time_step(spec, 0.1)
    bufs = [ud.clone(), torch.empty_like(ud), torch.empty_like(ud)]
    sol = one.rk_step(bufs, 0, 0.0, dt, 3)
    ref_rk = bufs[sol].cpu().numpy()

    meshes = [Mesh(spec, rank=r, nranks=P, xparts=xparts, vparts=vparts) for r in range(P)]
    assert sum(m.owned_dofs for m in meshes) == u.size
    parts = _split(spec, u, meshes)
    us = [torch.from_numpy(p).cuda() for p in parts]
    vs = [torch.empty_like(x) for x in us]
    apply_advection_group(meshes, us, vs)
    torch.cuda.synchronize()
    got_a = _join(spec, [v.cpu().numpy() for v in vs], meshes)
    assert np.array_equal(got_a, ref_a), f"{name}: A differs, max {np.nanmax(np.abs(got_a - ref_a)):.3e}"
    ora = oracle.apply_advection(spec, u)
    assert np.max(np.abs(got_a - ora)) <= 1e-12 * np.max(np.abs(ora))

    rb = [[x.clone(), torch.empty_like(x), torch.empty_like(x)] for x in us]
    sol = rk_step_group(meshes, rb, 0, 0.0, dt, 3)
    torch.cuda.synchronize()
    got_rk = _join(spec, [b[sol].cpu().numpy() for b in rb], meshes)
    assert np.array_equal(got_rk, ref_rk), f"{name}: RK differs, max {np.nanmax(np.abs(got_rk - ref_rk)):.3e}"


def test_partitioned_fill_matches_numpy():
    import torch
    cfg = configs.CONFIGS["5d"]
    spec = dict(cfg["spec"], cells=[6, 6, 6, 4, 4])
    seed = configs.seed_of("5d")
    u = inputs.full_vector(spec, cfg["recipe"], seed)
    meshes = [Mesh(spec, rank=r, nranks=8) for r in range(8)]
    parts = []
    for m in meshes:
        g = torch.empty(m.owned_dofs, dtype=torch.float64, device="cuda")
        m.fill_initial(g, cfg["recipe"], seed)
        parts.append(g.cpu().numpy())
    got = _join(spec, parts, meshes)
    assert np.max(np.abs(got - u)) <= 1e-14 * np.max(np.abs(u))


def test_multirank_single_calls_need_a_transport():
    import torch
    from paper_2002_08110_b200 import HDError
    spec = CASES[1][1]
    m = Mesh(spec, rank=0, nranks=2)
    x = torch.zeros(m.owned_dofs, dtype=torch.float64, device="cuda")
    with pytest.raises(HDError):
        m.apply_advection(x, torch.empty_like(x))
