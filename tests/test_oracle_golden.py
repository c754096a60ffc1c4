"""The oracle (oracle/panel_oracle.py) is pinned against the reference:
its factors match the reference's factor slabs (tests/golden/), and it
reproduces the reference's known-answer tests."""

import json
import os

import numpy as np
import pytest

from _cases import small_cases
from oracle import panel_oracle as O
from paper_1405_2636_b200 import sparse
from paper_1405_2636_b200.analysis import AnalyzeOptions, analyze
from paper_1405_2636_b200.errors import NotPositiveDefiniteError, SingularPivotError
from paper_1405_2636_b200.symbolic import allocate_panels, gather_factor

HERE = os.path.dirname(__file__)
SLABS = np.load(os.path.join(HERE, "golden", "factors_small.npz"))
GOLD = json.load(open(os.path.join(HERE, "golden", "golden.json")))


@pytest.mark.parametrize("name,A,form", list(small_cases()), ids=lambda x: x if isinstance(x, str) else "")
def test_oracle_matches_reference_factor(name, A, form):
    an = analyze(A, AnalyzeOptions(form=form))
    store = O.factor_analysis(an)
    ref = SLABS[name]
    assert store.slab.shape == ref.shape
    err = np.abs(store.slab - ref).max() / np.abs(ref).max()
    assert err <= 1e-13, err
    b = sparse.spmv(A, np.ones(A.n))
    x = O.solve(an.symbol, store, b, form, an.perm.perm)
    assert sparse.residual_norm(A, x, b) <= max(1e-13, 10 * GOLD["small"][name]["residual"])


def test_oracle_24_cube_sampled():
    g = GOLD["large"]["lap3d_24_llt"]
    an = analyze(sparse.gen_laplacian(3, (24, 24, 24)))
    store = O.factor_analysis(an)
    s = store.slab[::g["sample_step"]]
    assert np.abs(s - np.array(g["sample"])).max() / g["max_abs_L"] <= 1e-13


def test_oracle_unit_kats():
    # reference tests/test_kernels.py:29-33 ([[4,2],[2,3]] -> [[2,0],[1,sqrt2]])
    a = np.asfortranarray([[4.0, 0.0], [2.0, 3.0]])
    O.factor_panel(a, 0, "llt", 0.0)
    assert a[1, 0] == 1.0 and abs(a[1, 1] - np.sqrt(2)) <= 1e-15 and a[0, 0] == 2.0
    # LDLt [[2,2],[2,5]] -> L10 = 1, d = (2, 3)   (test_kernels.py:207-212)
    a = np.asfortranarray([[2.0, 0.0], [2.0, 5.0]])
    O.factor_panel(a, 0, "ldlt", 0.0)
    assert a[1, 0] == 1.0 and np.diagonal(a).tolist() == [2.0, 3.0]
    # grouped solve on stacked rows: panel [[2],[6],[8]] -> [[2],[3],[4]]
    a = np.asfortranarray([[4.0], [6.0], [8.0]])
    O.factor_panel(a, 0, "llt", 0.0)
    assert a[:, 0].tolist() == [2.0, 3.0, 4.0]


def test_oracle_failure_columns():
    a = np.asfortranarray([[1.0, 0.0], [2.0, 1.0]])
    with pytest.raises(NotPositiveDefiniteError) as e:
        O.factor_panel(a, 5, "llt", 0.0)
    assert e.value.column == 6
    a = np.asfortranarray([[0.0]])
    with pytest.raises(SingularPivotError) as e:
        O.factor_panel(a, 3, "ldlt", 1e-13)
    assert e.value.column == 3


def test_oracle_vs_dense_cholesky(rng):
    from conftest import rand_spd
    for _ in range(5):
        n = int(rng.integers(20, 120))
        A, _ = rand_spd(rng, n, 0.15)
        an = analyze(A)
        store = O.factor_analysis(an)
        L, _ = gather_factor(an.symbol, store)
        expect = np.linalg.cholesky(an.A_perm.to_dense())
        assert np.abs(L - expect).max() <= 1e-12 * np.abs(expect).max()


def test_host_allocate_matches_dense():
    A = sparse.gen_laplacian(2, (5, 4))
    an = analyze(A)
    store = allocate_panels(an.symbol, an.A_perm)
    L, _ = gather_factor(an.symbol, store)
    assert np.array_equal(L, np.tril(an.A_perm.to_dense()))
