"""CPU checks of the C ABI boundary (no compute calls without a GPU): the library loads, exports
every symbol include/hd.h declares, validates descriptors on the host, and its host-only tables
match the independent definitions."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2002_08110_b200 import _binding as B
from paper_2002_08110_b200 import build as hdbuild

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    hdbuild.build()
    return B.load_library()


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "hd.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(hd_[a-z0-9_]+)\s*\(", txt)))


def test_exports_every_declared_symbol(lib):
    syms = header_symbols()
    assert len(syms) >= 10
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(B.EXPORTS) == syms


def test_nm_shows_symbols_are_extern_c():
    import subprocess
    out = subprocess.check_output(["nm", "-D", "--defined-only", B.LIB_PATH]).decode()
    for s in header_symbols():
        assert re.search(rf"\bT {s}$", out, re.M), s


def _create(lib, spec, **kw):
    ds = B.make_desc(spec, **kw)
    h = ctypes.c_void_p()
    st = lib.hd_create_mesh(ctypes.byref(ds), ctypes.byref(h))
    return st, lib.hd_last_error().decode()


def _spec(**over):
    s = dict(d_x=1, d_v=1, k=3, cells=[4, 4], lo=[0, 0], hi=[1, 1], a_const=[1.0, 0.5],
             a_lin=[[0, 0], [0, 0]], flux="upwind")
    s.update(over)
    return s


def test_invalid_descriptors_are_rejected_on_host(lib):
    # invalid dim or zero subdivision -> construction error
    assert _create(lib, _spec(cells=[0, 4]))[0] == -1
    assert _create(lib, _spec(hi=[1, 0]))[0] == -1
    assert _create(lib, _spec(a_lin=[[1.0, 0], [0, 0]]))[0] == -1          # div a != 0
    st, msg = _create(lib, _spec(d_x=4, d_v=1, cells=[2] * 5, lo=[0] * 5, hi=[1] * 5, a_const=[1] * 5,
                                 a_lin=[[0] * 5] * 5))
    assert st == -1 and "d_x" in msg
    assert _create(lib, _spec(), rank=2, nranks=2)[0] == -1
    assert _create(lib, _spec(), rank=0, nranks=3)[0] == -1                 # 3 does not divide |C_x| = 4
    # valid but unsupported: central flux across ranks, k = 0, v = 0 inside a cell (upwind only, C11)
    # (a valid single-rank central mesh passes host validation: HD_OK on a GPU box, HD_ERR_CUDA here)
    assert _create(lib, _spec(flux="central"))[0] in (0, -3)
    assert _create(lib, _spec(flux="central"), rank=0, nranks=2)[0] == -2
    assert _create(lib, _spec(lo=[0, -1], hi=[1, 1], cells=[4, 3], a_const=[0.0, 0.3], a_lin=[[0, 1.0], [0, 0]],
                              flux="central"))[0] in (0, -3)
    assert _create(lib, _spec(k=0))[0] == -2
    st, msg = _create(lib, _spec(lo=[0, -1], hi=[1, 1], cells=[4, 3], a_const=[0.0, 0.3],
                                 a_lin=[[0, 1.0], [0, 0]]))
    assert st == -2 and "C11" in msg
    # overflow of 64-bit DoF indexing
    assert _create(lib, _spec(cells=[1 << 40, 1 << 20]))[0] == -1


def test_tables_match_independent_definitions(lib):
    for n in range(2, 7):
        t = B.tables_1d(n)
        x, w = np.polynomial.legendre.leggauss(n)
        x, w = 0.5 * (x + 1), 0.5 * w
        assert np.max(np.abs(t["xi"] - x)) < 1e-15
        assert np.max(np.abs(t["w"] - w)) < 1e-15
        # tau: Lagrange values at the faces; lam = +-tau(other face)/w
        V = np.vander(x, increasing=True)
        l0 = np.linalg.solve(V.T, np.array([0.0 ** p for p in range(n)]))
        l1 = np.linalg.solve(V.T, np.ones(n))
        assert np.max(np.abs(t["tau"][0] - l1)) < 1e-13
        assert np.max(np.abs(t["tau"][1] - l0)) < 1e-13
        assert np.max(np.abs(t["lam"][0] - l0 / w)) < 1e-12
        assert np.max(np.abs(t["lam"][1] + l1 / w)) < 1e-12
        # K applied to a constant line plus the lift of the same constant trace gives 0
        for s in range(2):
            assert np.max(np.abs(t["K"][s].sum(axis=1) + t["lam"][s])) < 1e-12


def test_tables_reproduce_1d_operator(lib):
    # assembling the periodic 1D operator from (K, lam, tau) equals the textbook 1D DG matrix of the
    # worked example (tests/golden/adv1d_k1_two_cells.txt) for n = 2, and is exact on polynomials
    from conftest import load_golden
    t = B.tables_1d(2)
    h = 0.5
    L = np.zeros((4, 4))
    for e in range(2):
        r = slice(2 * e, 2 * e + 2)
        L[r, r] += t["K"][0] / h
        en = (e - 1) % 2
        L[r, slice(2 * en, 2 * en + 2)] += np.outer(t["lam"][0], t["tau"][0]) / h
    exp = np.zeros((4, 4))
    for r_, c_, p, q in load_golden("adv1d_k1_two_cells.txt"):
        exp[int(r_), int(c_)] = float(p) + float(q) * np.sqrt(3.0)
    assert np.max(np.abs(L - exp)) < 1e-13


def test_lsrk_coefficients_order_conditions(lib):
    A, Bc = B.lsrk_coefficients()
    # rebuild the Butcher tableau of the 2N scheme (stage i evaluated at U_{i-1})
    def coef(j, upto):
        tot = 0.0
        for r in range(j, upto + 1):
            p = 1.0
            for l in range(j + 1, r + 1):
                p *= A[l]
            tot += Bc[r] * p
        return tot
    a = np.zeros((5, 5))
    for i in range(5):
        for j in range(i):
            a[i, j] = coef(j, i - 1)
    b = np.array([coef(j, 4) for j in range(5)])
    c = a.sum(axis=1)
    res = [b.sum() - 1, b @ c - 0.5, b @ c**2 - 1 / 3, b @ (a @ c) - 1 / 6, b @ c**3 - 0.25,
           b @ (c * (a @ c)) - 1 / 8, b @ (a @ c**2) - 1 / 12, b @ (a @ (a @ c)) - 1 / 24]
    assert np.max(np.abs(res)) < 1e-14
    assert A[0] == 0.0


def test_basis_tables_match_independent_definitions(lib):
    """GLL points against their closed forms and the four basis-change matrices against interpolation of
    monomials (T maps GLL-point values of x^p to Gauss-point values, p <= k) -- no oracle code involved."""
    from paper_2002_08110_b200._binding import basis_tables, tables_1d
    s5, s37 = np.sqrt(1 / 5), np.sqrt(3 / 7)
    closed = {2: [0, 1], 3: [0, 0.5, 1], 4: [0, (1 - s5) / 2, (1 + s5) / 2, 1], 5: [0, (1 - s37) / 2, 0.5, (1 + s37) / 2, 1]}
    for n in range(2, 7):
        gll, T = basis_tables(n)
        if n in closed:
            assert np.max(np.abs(gll - np.array(closed[n]))) < 1e-15
        assert np.all(np.diff(gll) > 0) and abs(gll[0]) < 1e-15 and abs(gll[-1] - 1) < 1e-15
        xg = tables_1d(n)["xi"]
        for p in range(n):
            assert np.max(np.abs(T[0] @ gll ** p - xg ** p)) < 1e-14
            assert np.max(np.abs(T[1] @ xg ** p - gll ** p)) < 1e-14
        assert np.array_equal(T[2], T[0].T) and np.array_equal(T[3], T[1].T)
        assert np.max(np.abs(T[0] @ T[1] - np.eye(n))) < 1e-13

