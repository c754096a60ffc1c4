"""The host analysis reproduces the reference's permutation and block symbol
exactly (digests from tests/golden/make_golden.py, which ran the reference)."""

import json
import os

import numpy as np
import pytest

from _cases import small_cases
from digest import array_symbol_digest
from paper_1405_2636_b200 import sparse
from paper_1405_2636_b200.analysis import AnalyzeOptions, analyze

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))


@pytest.mark.parametrize("name,A,form", list(small_cases()), ids=lambda x: x if isinstance(x, str) else "")
def test_small_symbols_identical(name, A, form):
    g = GOLD["small"][name]
    an = analyze(A, AnalyzeOptions(form=form))
    assert array_symbol_digest(an.symbol, an.perm.perm) == g["digest"]
    assert an.flops == g["flops"]


def test_lap3d_24_symbol_identical():
    g = GOLD["large"]["lap3d_24_llt"]
    an = analyze(sparse.gen_laplacian(3, (24, 24, 24)))
    assert array_symbol_digest(an.symbol, an.perm.perm) == g["digest"]
    assert (an.flops, an.symbol.nnz_l, an.symbol.npanels, an.symbol.block_count()) == \
        (g["flops"], g["nnz_l"], g["npanels"], g["nblocks"])


@pytest.mark.parametrize("N", [40, 60])
def test_lap3d_large_symbol_identical(N):
    g = GOLD["large"][f"lap3d_{N}_llt"]
    an = analyze(sparse.gen_laplacian(3, (N, N, N)))
    assert array_symbol_digest(an.symbol, an.perm.perm) == g["digest"]
    assert an.flops == g["flops"] == {40: 12359392298, 60: 159853212195}[N]


def test_ldlt_shift_symbol_identical():
    g = GOLD["large"]["lap3d_24_ldlt_shift"]
    A = sparse.shift_diagonal(sparse.gen_laplacian(3, (24, 24, 24)), 0.5)
    an = analyze(A, AnalyzeOptions(form="ldlt"))
    assert array_symbol_digest(an.symbol, an.perm.perm) == g["digest"]
    assert an.flops == g["flops"]


def test_cli_kat_2x1_grid():
    # reference tests/test_cli.py:35-40: factor --lap2d 2 1 -> nnz_l=3, flops=5
    an = analyze(sparse.gen_laplacian(2, (2, 1)))
    assert an.symbol.nnz_l == 3 and an.flops == 5


def test_laplacian_counts():
    # reference tests/test_sparse.py:147-150: 3D 4^3 lower nnz = 208
    assert sparse.gen_laplacian(3, (4, 4, 4)).nnz == 208


def test_dense_panel_flops():
    # reference tests/test_kernels.py:300-306: one dense 10x10 panel -> 385 flops
    rng = np.random.default_rng(20240211)
    from _cases import rand_spd
    A = rand_spd(rng, 10, 1.1)
    an = analyze(A, AnalyzeOptions(ordering="natural", amalgamation=0, split_width=0))
    assert an.symbol.npanels == 1 and an.flops == 385
