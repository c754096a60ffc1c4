"""LU (real, complex) and complex LLt / LDLt on the B200 engine vs the
extension oracle (oracle/panel_oracle_ext.py, pinned by
tests/test_oracle_ext.py to dense factorizations and scipy).

Tolerances: factor entries (L slab and the U^T slab) <= 1e-12 relative
(max|d|/max|ref|) - the kernels and the oracle differ only in summation
order on these well-conditioned matrices; backward error
||Ax-b||/||b|| <= 1e-12 (north star), through the GPU solve.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import panel_oracle_ext as X  # noqa: E402
from paper_1405_2636_b200 import sparse  # noqa: E402
from paper_1405_2636_b200.analysis import AnalyzeOptions, analyze  # noqa: E402
from paper_1405_2636_b200.errors import NotPositiveDefiniteError, SingularPivotError  # noqa: E402
from paper_1405_2636_b200.pipeline import factorize  # noqa: E402


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def cases(N):
    A = sparse.gen_convdiff27(N)
    Ac = sparse.gen_convdiff27(N, complex_shift=1.0)
    S = sparse.symmetrize_pattern(Ac)
    yield "lu", A, "lu"
    yield "lu_complex", Ac, "lu"
    yield "llt_complex", S, "llt"
    yield "ldlt_complex", S, "ldlt"
    yield "ldlt_complex_shift", sparse.shift_diagonal(S, 30.0), "ldlt"


@pytest.mark.parametrize("N", [6, 12])
def test_forms_match_oracle(N):
    for name, A, form in cases(N):
        an = analyze(A, AnalyzeOptions(form=form))
        res = factorize(an)
        st, ut = X.factor_analysis(an)
        assert res.store.slab.dtype == st.slab.dtype, name
        assert rel(res.store.slab, st.slab) <= 1e-12, name
        if form == "lu":
            assert rel(res.ustore.slab, ut.slab) <= 1e-12, name
        b = sparse.spmv(A, np.ones(A.n) * (1 + 0.5j if np.iscomplexobj(A.values) else 1.0))
        x = res.solve(b)
        assert sparse.backward_error(A, x, b) <= 1e-12, name


def test_lu_random_general_wide_panels():
    """Random sparse nonsymmetric matrices with wide panels (diagonal-block
    steps, TRSM items, trailing tiles of the wide-panel chain)."""
    rng = np.random.default_rng(31)
    for n, dens, cplx in ((300, 0.02, False), (300, 0.02, True), (700, 0.006, False)):
        mask = (rng.random((n, n)) < dens) & ~np.eye(n, dtype=bool)
        V = rng.uniform(-1, 1, (n, n)) * mask
        if cplx:
            V = V + 1j * rng.uniform(-1, 1, (n, n)) * mask
        V = V + np.diag(np.abs(V).sum(axis=1) + 1.0)
        r, c = np.nonzero(V)
        A = sparse.from_coo(n, r, c, V[r, c], sparse.GENERAL)
        an = analyze(A, AnalyzeOptions(form="lu"))
        assert an.symbol.max_width() > 64
        res = factorize(an)
        st, ut = X.factor_analysis(an)
        assert rel(res.store.slab, st.slab) <= 1e-12
        assert rel(res.ustore.slab, ut.slab) <= 1e-12
        b = V @ np.ones(n)
        assert sparse.backward_error(A, res.solve(b), b) <= 1e-12


def test_lu_deterministic_bitwise():
    A = sparse.gen_convdiff27(14, complex_shift=1.0)
    an = analyze(A, AnalyzeOptions(form="lu"))
    a = factorize(an).device_store.tensor.clone()
    b = factorize(an).device_store.tensor
    assert torch.equal(a, b)


def test_lu_singular_pivot_column():
    n = 6
    D = np.diag(np.arange(1.0, n + 1))
    D[:2, :2] = [[0.0, 1.0], [2.0, 0.0]]
    r, c = np.nonzero(D)
    A = sparse.from_coo(n, r, c, D[r, c], sparse.GENERAL)
    an = analyze(A, AnalyzeOptions(form="lu", ordering="natural"))
    with pytest.raises(SingularPivotError) as ei:
        factorize(an)
    assert ei.value.column == 0


def test_complex_llt_zero_pivot_column():
    A = sparse.from_coo(2, np.array([0, 1, 1]), np.array([0, 0, 1]),
                        np.array([1.0 + 0j, 1.0 + 0j, 1.0 + 0j]), sparse.SYMMETRIC_LOWER)
    an = analyze(A, AnalyzeOptions(form="llt", ordering="natural"))
    with pytest.raises(NotPositiveDefiniteError) as ei:
        factorize(an)
    assert ei.value.column == 1


@pytest.mark.slow
@pytest.mark.parametrize("cplx", [False, True])
def test_lu_convdiff80_backward_error(cplx):
    """BASELINE configs[3]: LU of the 27-point convection-diffusion 80^3
    (real and complex); backward error <= 1e-12 through the GPU solve."""
    A = sparse.gen_convdiff27(80, complex_shift=1.0 if cplx else None)
    an = analyze(A, AnalyzeOptions(form="lu"))
    res = factorize(an, download=False)
    b = sparse.spmv(A, np.ones(A.n) * (1 + 0.5j if cplx else 1.0))
    assert sparse.backward_error(A, res.solve(b), b) <= 1e-12
