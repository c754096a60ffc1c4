"""Host-side pipeline helpers (CPU): the pivot threshold of the reference
(kernels.py:32-40, recomputed from the current values on every
factorize, pipeline.py:88-91) with its cached diagonal positions."""
import numpy as np

from paper_1405_2636_b200 import sparse
from paper_1405_2636_b200.analysis import analyze
from paper_1405_2636_b200.pipeline import default_pivot_threshold, diagonal_positions


def _reference_threshold(A):
    on = A.rowidx == A.entry_cols()
    return 1e-13 * float(np.abs(A.values[on]).max()) if on.any() else 0.0


def test_threshold_matches_reference_formula():
    for A in (sparse.gen_laplacian(2, (16, 16)), sparse.gen_laplacian(3, (6, 6, 6)),
              sparse.shift_diagonal(sparse.gen_laplacian(3, (5, 5, 5)), 0.5)):
        an = analyze(A)
        assert default_pivot_threshold(an.A_perm) == _reference_threshold(an.A_perm)


def test_threshold_follows_in_place_value_changes():
    an = analyze(sparse.gen_laplacian(3, (6, 6, 6)))
    A = an.A_perm
    t0 = default_pivot_threshold(A)
    pos = diagonal_positions(A)
    assert diagonal_positions(A) is pos  # cached per pattern
    A.values[pos[3]] = 1e6  # same pattern, new values: recomputed from them
    assert default_pivot_threshold(A) == 1e-13 * 1e6 != t0
    assert default_pivot_threshold(A) == _reference_threshold(A)


def test_threshold_positions_per_pattern():
    a1 = analyze(sparse.gen_laplacian(2, (8, 8))).A_perm
    a2 = analyze(sparse.gen_laplacian(2, (9, 9))).A_perm
    p1, p2 = diagonal_positions(a1), diagonal_positions(a2)
    assert len(p1) == a1.n and len(p2) == a2.n
    assert np.array_equal(a1.rowidx[p1], a1.entry_cols()[p1])
    assert np.array_equal(a2.rowidx[p2], a2.entry_cols()[p2])
