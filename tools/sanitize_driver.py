"""Small invocations of every kernel path for compute-sanitizer (memcheck / racecheck / synccheck):
pencil mode with published traces and in-group neighbours (5D, CT = 4), pencil mode with CT = 2 (6D n = 2),
multi-pencil groups (3D), degenerate meshes (one cell along some dims), multi-rank halo (loopback), each
through apply_advection, inverse mass and two LSRK steps.

python tools/sanitize_driver.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2002_08110_b200 import Mesh, configs  # noqa: E402
from paper_2002_08110_b200._binding import apply_advection_group, rk_step_group  # noqa: E402


def spec(d_x, d_v, k, cells, vlasov=True):
    d = d_x + d_v
    lo = [0.0] * d_x + [-1.5] * d_v
    hi = [1.0] * d_x + [1.5] * d_v
    a_const = [0.7, -0.4, 0.5][:d_x] + [0.3, -0.2, 0.1][:d_v]
    a_lin = [[0.0] * d for _ in range(d)]
    if vlasov:
        for i in range(min(d_x, d_v)):
            a_lin[i][d_x + i] = 1.0
            a_const[i] = 0.0
    return dict(d_x=d_x, d_v=d_v, k=k, cells=list(cells), lo=lo, hi=hi, a_const=a_const, a_lin=a_lin,
                flux="upwind")


CASES = [
    ("5d-pencil-ct4", spec(3, 2, 3, [6, 4, 2, 2, 2])),
    ("6d-n2-pencil-ct2", spec(3, 3, 1, [20, 2, 2, 2, 2, 2])),
    ("3d-multipencil", spec(2, 1, 2, [3, 2, 2])),
    ("4d-degenerate", spec(2, 2, 3, [1, 1, 2, 2])),
    ("2d-const", spec(1, 1, 3, [8, 8], vlasov=False)),
]


def run(name, sp):
    m = Mesh(sp)
    N = m.owned_dofs
    u = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, N)).cuda()
    v = torch.empty_like(u)
    m.apply_advection(u, v)
    m.apply_inv_mass(v)
    bufs = [u.clone(), torch.empty_like(u), torch.empty_like(u)]
    sol = m.rk_step(bufs, 0, 0.0, 1e-3, 2)
    torch.cuda.synchronize()
    print(name, "ok", float(bufs[sol].abs().sum()))
    m.close()


def run_group():
    sp = spec(3, 2, 3, [6, 4, 2, 2, 2])
    P = 2
    ms = [Mesh(sp, rank=r, nranks=P) for r in range(P)]
    us = [torch.from_numpy(np.random.default_rng(r).uniform(-1, 1, m.owned_dofs)).cuda() for r, m in enumerate(ms)]
    vs = [torch.empty_like(x) for x in us]
    apply_advection_group(ms, us, vs)
    bufs = [[x.clone(), torch.empty_like(x), torch.empty_like(x)] for x in us]
    rk_step_group(ms, bufs, 0, 0.0, 1e-3, 1)
    torch.cuda.synchronize()
    print("5d-group-P2 ok")


if __name__ == "__main__":
    for name, sp in CASES:
        run(name, sp)
    run_group()
