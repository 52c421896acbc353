"""Vlasov-Poisson measurements (NEXT-1): the Landau-damping run (1x1v, kappa = 0.5, alpha = 0.01) with the
fitted damping rate / frequency against the dispersion root, and the device time of one coupled LSRK stage
(rho, Poisson/E, FCL operator with a = (v, -E), M^-1, 2N update) on a 2x2v mesh of the 4D config's size
(16^4 cells, k = 3, 16.8M DoFs). One JSON line.

python tools/vp_run.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import capi, vp  # noqa: E402
from paper_2002_08110_b200 import Mesh  # noqa: E402
from test_oracle_vp import vp_spec  # noqa: E402


def landau(kap=0.5, alpha=0.01, cells=(16, 32), T=30.0, dt=0.01, every=5):
    spec = vp_spec(1, 3, list(cells), [2 * np.pi / kap], 6.0)
    m = Mesh(spec)
    n = 4
    xi, _ = capi.gauss_legendre(n)
    cx, cv = spec["cells"]
    hx, hv = 2 * np.pi / kap / cx, 12.0 / cv
    X = (np.arange(cx)[:, None] + xi[None, :]) * hx
    V = -6.0 + (np.arange(cv)[:, None] + xi[None, :]) * hv
    f0 = ((1 + alpha * np.cos(kap * X))[None, :, None, :] *
          (np.exp(-V**2 / 2) / np.sqrt(2 * np.pi))[:, None, :, None]).reshape(-1)
    N = m.owned_dofs
    bufs = [torch.from_numpy(f0).cuda(), torch.empty(N, dtype=torch.float64, device="cuda"),
            torch.empty(N, dtype=torch.float64, device="cuda")]
    E = torch.empty(m.vp_sizes()[1], dtype=torch.float64, device="cuda")
    ts, en = [], []
    t = 0.0
    while t < T - 1e-9:
        m.vp_fields(bufs[0], None, E)
        torch.cuda.synchronize()
        ts.append(t)
        en.append(vp.field_energy(spec, E.cpu().numpy()))
        m.vp_rk_step(bufs, t, dt, every)
        t += dt * every
    ts, en = np.array(ts), np.array(en)
    pk = [i for i in range(1, len(en) - 1) if en[i] > en[i - 1] and en[i] >= en[i + 1] and ts[i] > 1.5]
    slope = float(np.polyfit(ts[pk], np.log(en[pk]), 1)[0])
    om = vp.landau_root(kap)
    return {"kappa": kap, "alpha": alpha, "cells": list(cells), "k": 3, "dt": dt, "T": T,
            "gamma_fit": slope / 2, "gamma_root": om.imag, "omega_fit": float(np.pi / np.mean(np.diff(ts[pk]))),
            "omega_root": om.real, "peaks": [float(ts[i]) for i in pk],
            "energy_first_last": [float(en[0]), float(en[-1])]}


def stage_rate(reps=10):
    spec = vp_spec(2, 3, [16, 16, 16, 16], [4 * np.pi, 4 * np.pi], 6.0)
    m = Mesh(spec)
    N = m.owned_dofs
    rng = np.random.default_rng(1)
    f = torch.from_numpy(0.1 + 0.01 * rng.uniform(-1, 1, N)).cuda()
    bufs = [f, torch.empty_like(f), torch.empty_like(f)]
    s = torch.cuda.current_stream()
    m.vp_rk_step(bufs, 0.0, 1e-3, 1, s)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    m.vp_rk_step(bufs, 0.0, 1e-3, reps, s)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / (5 * reps)
    return {"mesh": "2x2v 16^4 cells k=3", "dofs": N, "ms_per_stage": ms, "gdofs_per_stage": N / (ms * 1e-3) / 1e9,
            "launches_per_stage": 8}


if __name__ == "__main__":
    if "--stage-only" in sys.argv:
        print(json.dumps({"vp_stage_4d": stage_rate(reps=1)}))
    else:
        print(json.dumps({"landau": landau(), "vp_stage_4d": stage_rate()}))
