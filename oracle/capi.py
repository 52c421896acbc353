"""ctypes binding of the O2 oracle (``hd_oracle.cpp``). TEST INFRASTRUCTURE ONLY.

A mesh spec is a plain dict::

    {"d_x": int, "d_v": int, "k": int, "cells": [..d ints..], "lo": [..], "hi": [..],
     "a_const": [..d..], "a_lin": [[..d..]..d..] (optional), "flux": "upwind"|"central"}

Global DoF order (reading C19): g = cell * n^d + sum_i m_i n^i, cell =
sum_i c_i prod_{j<i} cells_j (first axis fastest, x dims before v dims).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "hd_oracle.cpp")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


class OrDesc(ctypes.Structure):
    _fields_ = [
        ("d_x", ctypes.c_int),
        ("d_v", ctypes.c_int),
        ("k", ctypes.c_int),
        ("cells", ctypes.c_longlong * 6),
        ("lo", ctypes.c_double * 6),
        ("hi", ctypes.c_double * 6),
        ("a_const", ctypes.c_double * 6),
        ("a_lin", ctypes.c_double * 36),
        ("flux", ctypes.c_int),
    ]


def build(force: bool = False) -> str:
    """Compile liboracle.so (g++ -O2 -fopenmp). Building the checker is not using it."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["g++", "-O2", "-fopenmp", "-shared", "-fPIC", "-o", tmp, _SRC])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.POINTER
        d = ctypes.c_double
        _lib.or_apply_advection.argtypes = [P(OrDesc), P(d), P(d), ctypes.c_int]
        _lib.or_apply_advection_cells.argtypes = [P(OrDesc), ctypes.c_longlong, P(ctypes.c_longlong), P(d), P(d),
                                                  ctypes.c_int]
        _lib.or_apply_inv_mass.argtypes = [P(OrDesc), P(d)]
        _lib.or_apply_mass.argtypes = [P(OrDesc), P(d)]
        _lib.or_rk_steps.argtypes = [P(OrDesc), P(d), P(d), P(d), d, d, ctypes.c_int]
        _lib.or_dof_count.argtypes = [P(OrDesc)]
        _lib.or_dof_count.restype = ctypes.c_longlong
        _lib.or_gauss_legendre.argtypes = [ctypes.c_int, P(d), P(d)]
        _lib.or_lagrange_eval.argtypes = [ctypes.c_int, d, P(d), P(d)]
        _lib.or_rk_coefficients.argtypes = [P(d), P(d), P(d)]
        _lib.or_numerical_flux.argtypes = [d, d, d, ctypes.c_int]
        _lib.or_numerical_flux.restype = d
    return _lib


def desc(spec: dict) -> OrDesc:
    ds = OrDesc()
    d = spec["d_x"] + spec["d_v"]
    ds.d_x, ds.d_v, ds.k = spec["d_x"], spec["d_v"], spec["k"]
    for i in range(d):
        ds.cells[i] = int(spec["cells"][i])
        ds.lo[i] = float(spec["lo"][i])
        ds.hi[i] = float(spec["hi"][i])
        ds.a_const[i] = float(spec["a_const"][i])
        if spec.get("a_lin") is not None:
            for j in range(d):
                ds.a_lin[6 * i + j] = float(spec["a_lin"][i][j])
    ds.flux = {"upwind": 0, "central": 1}[spec.get("flux", "upwind")]
    return ds


def _ptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def dof_count(spec: dict) -> int:
    n = lib().or_dof_count(ctypes.byref(desc(spec)))
    if n < 0:
        raise ValueError("invalid mesh spec")
    return int(n)


def apply_advection(spec: dict, u: np.ndarray, merged: bool = False) -> np.ndarray:
    """v = A(u) (weak form, reading C5) or M^-1 A(u) if merged."""
    u = np.ascontiguousarray(u, dtype=np.float64)
    v = np.empty_like(u)
    rc = lib().or_apply_advection(ctypes.byref(desc(spec)), _ptr(u), _ptr(v), int(merged))
    if rc:
        raise ValueError("or_apply_advection failed")
    return v


def apply_advection_cells(spec: dict, cell_ids: np.ndarray, u_cells: np.ndarray, merged: bool = False) -> np.ndarray:
    """Per-cell A for sampled parity: u_cells[c] = [own, dim0-left, dim0-right, dim1-left, ...]."""
    cell_ids = np.ascontiguousarray(cell_ids, dtype=np.int64)
    u_cells = np.ascontiguousarray(u_cells, dtype=np.float64)
    nc = cell_ids.shape[0]
    out = np.empty((nc, u_cells.shape[-1]), dtype=np.float64)
    rc = lib().or_apply_advection_cells(ctypes.byref(desc(spec)), nc,
                                        cell_ids.ctypes.data_as(ctypes.POINTER(ctypes.c_longlong)),
                                        _ptr(u_cells), _ptr(out), int(merged))
    if rc:
        raise ValueError("or_apply_advection_cells failed")
    return out


def apply_inv_mass(spec: dict, u: np.ndarray) -> np.ndarray:
    v = np.array(u, dtype=np.float64, copy=True)
    if lib().or_apply_inv_mass(ctypes.byref(desc(spec)), _ptr(v)):
        raise ValueError("or_apply_inv_mass failed")
    return v


def apply_mass(spec: dict, u: np.ndarray) -> np.ndarray:
    v = np.array(u, dtype=np.float64, copy=True)
    if lib().or_apply_mass(ctypes.byref(desc(spec)), _ptr(v)):
        raise ValueError("or_apply_mass failed")
    return v


def rk_steps(spec: dict, u: np.ndarray, t: float, dt: float, nsteps: int) -> np.ndarray:
    v = np.array(u, dtype=np.float64, copy=True)
    du = np.zeros_like(v)
    r = np.zeros_like(v)
    if lib().or_rk_steps(ctypes.byref(desc(spec)), _ptr(v), _ptr(du), _ptr(r), float(t), float(dt), int(nsteps)):
        raise ValueError("or_rk_steps failed")
    return v


def gauss_legendre(n: int):
    x = np.zeros(n)
    w = np.zeros(n)
    if lib().or_gauss_legendre(n, _ptr(x), _ptr(w)):
        raise ValueError("bad n")
    return x, w


def lagrange_eval(n: int, t: float):
    val = np.zeros(n)
    der = np.zeros(n)
    lib().or_lagrange_eval(n, float(t), _ptr(val), _ptr(der))
    return val, der


def rk_coefficients():
    a, b, c = np.zeros(5), np.zeros(5), np.zeros(5)
    lib().or_rk_coefficients(_ptr(a), _ptr(b), _ptr(c))
    return a, b, c


def numerical_flux(um: float, up: float, an: float, kind: str = "upwind") -> float:
    return lib().or_numerical_flux(um, up, an, {"upwind": 0, "central": 1}[kind])


def num_threads() -> int:
    return int(lib().or_num_threads())
