"""Run with the HD_DEBUG build of libhd.so (HD_LIB_PATH=.../libhd_debug.so): the device-side checks
(index bounds, halo freshness S:481, non-finite values after an RK stage S:508) stay silent on valid runs
of every kernel path the bench configs use, and a non-finite input is reported as HD_ERR_STATE.
Prints one line per case and 'DEBUG-CHECKS OK' at the end; exit 1 on a failure."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2002_08110_b200 import Mesh, apply_advection_group, rk_step_group  # noqa: E402
from paper_2002_08110_b200._binding import HDError  # noqa: E402


def spec(d_x, d_v, k, cells):
    d = d_x + d_v
    lin = [[0.0] * d for _ in range(d)]
    for i in range(min(d_x, d_v)):
        lin[i][d_x + i] = 1.0
    ac = [0.0] * d_x + [0.3, -0.2, 0.1][:d_v]
    if d_x > d_v:
        ac[d_x - 1] = 0.5
    return dict(d_x=d_x, d_v=d_v, k=k, cells=list(cells), lo=[0.0] * d_x + [-2.0] * d_v, hi=[1.0] * d_x + [2.0] * d_v,
                a_const=ac, a_lin=lin, flux="upwind")


def main():
    assert "debug" in os.environ.get("HD_LIB_PATH", ""), "run with HD_LIB_PATH=<libhd_debug.so>"
    ok = True
    cases = [("5d-pencil", spec(3, 2, 3, [6, 8, 4, 4, 4])), ("6d-pencil", spec(3, 3, 3, [4, 4, 4, 2, 2, 2])),
             ("4d-multipencil", spec(2, 2, 3, [4, 6, 2, 4]))]
    for name, sp in cases:
        m = Mesh(sp)
        u = torch.from_numpy(np.random.default_rng(3).uniform(-1, 1, m.owned_dofs)).cuda()
        v = torch.empty_like(u)
        m.apply_advection(u, v)
        bufs = [u.clone(), torch.empty_like(u), torch.empty_like(u)]
        m.rk_step(bufs, 0, 0.0, 1e-3, 2)
        print(name, "clean")
        # a non-finite value must be reported after the stage
        bad = u.clone()
        bad[m.owned_dofs // 2] = float("nan")
        bufs = [bad, torch.empty_like(u), torch.empty_like(u)]
        try:
            m.rk_step(bufs, 0, 0.0, 1e-3, 1)
            print(name, "NaN NOT reported")
            ok = False
        except HDError as e:
            ok = ok and "S:508" in str(e)
            print(name, "NaN reported:", e)
        m.close()
    # multi-rank loopback (halo freshness tags travel with the traces)
    for P in (2, 4):
        sp = spec(3, 2, 3, [6, 8, 4, 4, 4])
        ms = [Mesh(sp, rank=r, nranks=P) for r in range(P)]
        us = [torch.from_numpy(np.random.default_rng(r).uniform(-1, 1, x.owned_dofs)).cuda() for r, x in enumerate(ms)]
        vs = [torch.empty_like(x) for x in us]
        apply_advection_group(ms, us, vs)
        bufs = [[x.clone(), torch.empty_like(x), torch.empty_like(x)] for x in us]
        rk_step_group(ms, bufs, 0, 0.0, 1e-3, 2)
        print(f"5d-group-P{P} clean")
    print("DEBUG-CHECKS OK" if ok else "DEBUG-CHECKS FAILED")
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
