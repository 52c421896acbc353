"""Seeded synthetic inputs (reading C14). Holds none of the method's arithmetic.

Counter-based: the value at global DoF g depends only on (seed, g), so any subset of
cells can be regenerated independently (sampled parity at 6D) and the device-side
generator ``hd_fill_initial`` (csrc/hd_kernels.cu fill_kernel) implements the same recipe for
configs whose vectors do not fit host memory comfortably. Node positions use
``numpy.polynomial.legendre.leggauss`` (a library routine).

Recipes (value at node z, U = uniform[0,1) from splitmix64(g + seed * 2^40)):
  gauss2d    exp(-|z - (0.5, 0.5)|^2 / 0.02) + (2U - 1) 1e-3
  uniform    2U - 1
  sines      prod_i sin(2 pi z_i) + (2U - 1) 1e-3
  maxwellian (1 + 0.01 cos(0.5 x_1)) (2 pi)^(-d_v/2) exp(-|v|^2 / 2) (1 + (2U - 1) 1e-3)
"""
from __future__ import annotations

import numpy as np

RECIPES = {"gauss2d": 0, "uniform": 1, "sines": 2, "maxwellian": 3}

_M1 = np.uint64(0x9E3779B97F4A7C15)
_M2 = np.uint64(0xBF58476D1CE4E5B9)
_M3 = np.uint64(0x94D049BB133111EB)


def splitmix64(x: np.ndarray) -> np.ndarray:
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + _M1
        z = (z ^ (z >> np.uint64(30))) * _M2
        z = (z ^ (z >> np.uint64(27))) * _M3
        z = z ^ (z >> np.uint64(31))
    return z


def uniform01(seed: int, idx: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        x = np.asarray(idx, dtype=np.uint64) + (np.uint64(seed) << np.uint64(40))
    return (splitmix64(x) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def _nodes(n):
    x, _ = np.polynomial.legendre.leggauss(n)
    return 0.5 * (x + 1.0)


def cell_values(spec: dict, recipe: str, seed: int, cell_ids: np.ndarray, chunk: int = 1 << 22) -> np.ndarray:
    """Nodal values for the given global cell ids: array [len(cell_ids), n^d] (computed in chunks of
    about ``chunk`` values to bound temporary memory)."""
    d = spec["d_x"] + spec["d_v"]
    nd = (spec["k"] + 1) ** d
    cell_ids = np.asarray(cell_ids, dtype=np.int64).reshape(-1)
    per = max(1, chunk // nd)
    if len(cell_ids) <= per:
        return _cell_values(spec, recipe, seed, cell_ids)
    out = np.empty((len(cell_ids), nd))
    for s in range(0, len(cell_ids), per):
        out[s:s + per] = _cell_values(spec, recipe, seed, cell_ids[s:s + per])
    return out


def _cell_values(spec: dict, recipe: str, seed: int, cell_ids: np.ndarray) -> np.ndarray:
    d = spec["d_x"] + spec["d_v"]
    d_x = spec["d_x"]
    n = spec["k"] + 1
    nd = n ** d
    cells = np.array(spec["cells"], dtype=np.int64)
    lo = np.array(spec["lo"], float)
    h = (np.array(spec["hi"], float) - lo) / cells
    xi = _nodes(n)
    cell_ids = np.asarray(cell_ids, dtype=np.int64).reshape(-1)
    # cell coordinates (first axis fastest, reading C19)
    cc = np.empty((len(cell_ids), d), dtype=np.int64)
    r = cell_ids.copy()
    for i in range(d):
        cc[:, i] = r % cells[i]
        r //= cells[i]
    m = np.arange(nd, dtype=np.int64)
    mi = np.empty((nd, d), dtype=np.int64)
    rm = m.copy()
    for i in range(d):
        mi[:, i] = rm % n
        rm //= n
    # z[c, q, i]
    z = lo[None, None, :] + (cc[:, None, :].astype(float) + xi[mi][None, :, :]) * h[None, None, :]
    g = cell_ids[:, None] * nd + m[None, :]
    U = uniform01(seed, g)
    if recipe == "gauss2d":
        val = np.exp(-((z[..., 0] - 0.5) ** 2 + (z[..., 1] - 0.5) ** 2) / 0.02) + (2.0 * U - 1.0) * 1e-3
    elif recipe == "uniform":
        val = 2.0 * U - 1.0
    elif recipe == "sines":
        val = np.prod(np.sin(2.0 * np.pi * z), axis=-1) + (2.0 * U - 1.0) * 1e-3
    elif recipe == "maxwellian":
        v2 = np.sum(z[..., d_x:] ** 2, axis=-1)
        d_v = d - d_x
        val = ((1.0 + 0.01 * np.cos(0.5 * z[..., 0])) * (2.0 * np.pi) ** (-0.5 * d_v) * np.exp(-0.5 * v2)
               * (1.0 + (2.0 * U - 1.0) * 1e-3))
    else:
        raise ValueError(recipe)
    return val


def full_vector(spec: dict, recipe: str, seed: int) -> np.ndarray:
    ncell = int(np.prod(spec["cells"], dtype=np.int64))
    return cell_values(spec, recipe, seed, np.arange(ncell)).reshape(-1)


def neighbour_ids(spec: dict, cell_ids: np.ndarray) -> np.ndarray:
    """[len, 2d] periodic face neighbours (dim 0 left, dim 0 right, dim 1 left, ...)."""
    d = spec["d_x"] + spec["d_v"]
    cells = np.array(spec["cells"], dtype=np.int64)
    cell_ids = np.asarray(cell_ids, dtype=np.int64).reshape(-1)
    cc = np.empty((len(cell_ids), d), dtype=np.int64)
    r = cell_ids.copy()
    for i in range(d):
        cc[:, i] = r % cells[i]
        r //= cells[i]
    strides = np.concatenate([[1], np.cumprod(cells)[:-1]])
    out = np.empty((len(cell_ids), 2 * d), dtype=np.int64)
    for i in range(d):
        for s, off in ((0, -1), (1, 1)):
            cn = cc.copy()
            cn[:, i] = (cc[:, i] + off) % cells[i]
            out[:, 2 * i + s] = cn @ strides
    return out
