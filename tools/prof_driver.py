"""Small driver for ncu / compute-sanitizer runs: a few applications of one operator on one config.

python tools/prof_driver.py --config 5d --op rk --reps 3
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2002_08110_b200 import Mesh, configs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="5d")
ap.add_argument("--op", default="rk", choices=["rk", "adv", "mass", "fcl", "basis"])
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--cells", default=None, help="override cells, comma separated")
ap.add_argument("--time", action="store_true", help="print ms per application (CUDA events, after the reps as warm-up)")
a = ap.parse_args()
cfg = configs.CONFIGS[a.config]
spec = dict(cfg["spec"])
if a.cells:
    spec["cells"] = [int(x) for x in a.cells.split(",")]
m = Mesh(spec)
N = m.owned_dofs
bufs = [torch.empty(N, dtype=torch.float64, device="cuda") for _ in range(3)]
m.fill_initial(bufs[0], cfg["recipe"], configs.seed_of(a.config))
dt = configs.time_step(spec, cfg["cfl"])
sol = 0
for _ in range(a.reps):
    if a.op == "rk":
        sol = m.rk_step(bufs, sol, 0.0, dt, 1)
    elif a.op == "adv":
        m.apply_advection(bufs[0], bufs[1])
    elif a.op == "basis":
        m.basis_change(bufs[0], bufs[1], "gll_to_gauss")
    elif a.op == "fcl":
        m.apply_advection_fcl(bufs[0], bufs[1])
    else:
        m.apply_inv_mass(bufs[0])
torch.cuda.synchronize()
if a.time:
    fn = {"adv": lambda: m.apply_advection(bufs[0], bufs[1]), "mass": lambda: m.apply_inv_mass(bufs[0]),
          "basis": lambda: m.basis_change(bufs[0], bufs[1], "gll_to_gauss"),
          "fcl": lambda: m.apply_advection_fcl(bufs[0], bufs[1])}.get(a.op)
    if fn is not None:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print(f"{a.config} {a.op}: {ms:.3f} ms, {N / ms / 1e6:.1f} GDoF/s, {16 * N / ms / 1e6:.0f} GB/s at 16 B/DoF")
print("ok", N, float(bufs[sol][:1000].sum()))
