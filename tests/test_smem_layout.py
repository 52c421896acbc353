"""The padded shared-memory cell layout of the tile kernel (hd_cell.cuh cell_strides): every table entry
is injective (no two elements of a cell share a slot), keeps 16-byte pairs along dim 0 aligned when
N is even, grows a cell by at most 20 %, and is at least as bank-conflict free as the XOR swizzle it
replaced under the wavefront model of tools/smem_layout.py."""
import itertools
import os
import re
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import smem_layout as L  # noqa: E402


def table():
    src = open(os.path.join(ROOT, "paper_2002_08110_b200", "csrc", "hd_cell.cuh")).read()
    out = {}
    for d, n, body in re.findall(r"D == (\d) && N == (\d)\) return \{\{([0-9, ]+)\}\}", src):
        out[(int(d), int(n))] = [int(v) for v in body.split(",")]
    return out


TABLE = table()


def strides(D, N):
    return TABLE.get((D, N), [N ** i for i in range(D)])


def test_table_present():
    assert (6, 4) in TABLE and (5, 4) in TABLE and (4, 4) in TABLE


@pytest.mark.parametrize("D,N", list(L.built()))
def test_layout_injective_aligned_bounded(D, N):
    S = strides(D, N)
    assert len(S) == D and S[0] == 1
    pos = set()
    for digits in itertools.product(range(N), repeat=D):
        pos.add(sum(d * s for d, s in zip(digits, S)))
    assert len(pos) == N ** D, "two elements share a slot"
    if N % 2 == 0:
        assert all(s % 2 == 0 for s in S[1:]), "16-byte pairs along dim 0 must stay aligned"
    assert L.size_of(S, N) <= 1.2 * N ** D + 1


@pytest.mark.parametrize("D,N", list(L.built()))
def test_layout_no_more_conflicts_than_xor(D, N):
    S = strides(D, N)
    base = [N ** i for i in range(D)]
    assert L.cost(S, D, N) <= L.cost(base, D, N, phys=L.xor_phys(D, N)) + 1e-9


def test_search_reproduces_table():
    for (D, N), S in TABLE.items():
        assert L.search(D, N) == S
