"""The five synthetic workloads of BASELINE.json, as mesh specs.

A mesh spec is a plain dict (the same dict is accepted by the product binding and
by the test oracle): d_x, d_v, k, cells[d], lo[d], hi[d], a_const[d], a_lin[d][d],
flux. The advection field is a_i(z) = a_const[i] + sum_j a_lin[i][j] z_j
(Vlasov-like rows: a_lin[i][d_x+i] = 1, reading C10). Readings C8/C9: 3D/4D live on
[0,1]^d; the 5D/6D velocity box [-6,6]^d_v is periodic like every other dim.
"""
from __future__ import annotations

import math

import numpy as np


def _spec(d_x, d_v, k, cells, lo, hi, a_const, a_lin=None, flux="upwind"):
    d = d_x + d_v
    if a_lin is None:
        a_lin = [[0.0] * d for _ in range(d)]
    return dict(d_x=d_x, d_v=d_v, k=k, cells=list(cells), lo=list(lo), hi=list(hi), a_const=list(a_const),
                a_lin=[list(r) for r in a_lin], flux=flux)


def _vlasov_lin(d_x, d_v):
    d = d_x + d_v
    lin = [[0.0] * d for _ in range(d)]
    for i in range(min(d_x, d_v)):
        lin[i][d_x + i] = 1.0  # a_{x_i} = v_i (5D: x_3 keeps the constant 0.5, reading C10)
    return lin


FOUR_PI = 4.0 * math.pi

CONFIGS = {
    "2d": dict(index=0, recipe="gauss2d", cfl=0.1,
               spec=_spec(1, 1, 3, [8, 8], [0, 0], [1, 1], [1.0, 0.5])),
    "3d": dict(index=1, recipe="uniform", cfl=0.1,
               spec=_spec(2, 1, 4, [32] * 3, [0] * 3, [1] * 3, [1.0, 0.7, -0.3])),
    "4d": dict(index=2, recipe="sines", cfl=0.1,
               spec=_spec(2, 2, 3, [16] * 4, [0] * 4, [1] * 4, [1.0, 0.5, -0.25, 0.75])),
    "5d": dict(index=3, recipe="maxwellian", cfl=0.1,
               spec=_spec(3, 2, 3, [12] * 5, [0] * 3 + [-6] * 2, [FOUR_PI] * 3 + [6] * 2,
                          [0.0, 0.0, 0.5, 0.3, -0.2], _vlasov_lin(3, 2))),
    "6d": dict(index=4, recipe="maxwellian", cfl=0.1,
               spec=_spec(3, 3, 3, [10] * 6, [0] * 3 + [-6] * 3, [FOUR_PI] * 3 + [6] * 3,
                          [0.0, 0.0, 0.0, 0.3, -0.2, 0.1], _vlasov_lin(3, 3))),
}


def seed_of(name: str) -> int:
    """Reading C14: seed = 1000 * (config index) + 7."""
    return 1000 * CONFIGS[name]["index"] + 7


def dof_count(spec: dict) -> int:
    d = spec["d_x"] + spec["d_v"]
    return int(np.prod(spec["cells"], dtype=np.int64)) * (spec["k"] + 1) ** d


def max_speed(spec: dict, i: int) -> float:
    """max over the box of |a_i(z)| for the affine field (corners)."""
    d = spec["d_x"] + spec["d_v"]
    best = 0.0
    for corner in range(1 << d):
        z = [spec["hi"][j] if (corner >> j) & 1 else spec["lo"][j] for j in range(d)]
        a = spec["a_const"][i] + sum(spec["a_lin"][i][j] * z[j] for j in range(d))
        best = max(best, abs(a))
    return best


def time_step(spec: dict, cfl: float = 0.1) -> float:
    """Reading C12: dt = CFL / [(k+1)^2 sum_i max|a_i| / h_i]."""
    d = spec["d_x"] + spec["d_v"]
    s = 0.0
    for i in range(d):
        h = (spec["hi"][i] - spec["lo"][i]) / spec["cells"][i]
        s += max_speed(spec, i) / h
    return cfl / ((spec["k"] + 1) ** 2 * s)
