"""Pin the LU / complex oracle (oracle/panel_oracle_ext.py) - CPU only.

The reference factors only real LLt / LDLt (kernels.py:19-22), so the LU
and complex restatement is pinned against
  * dense no-pivot Doolittle LU / LDLt / Cholesky of the same permuted
    matrix (written directly in numpy, no supernodes),
  * the real oracle (oracle/panel_oracle.py, itself pinned to the
    reference's factors) on real symmetric input: complex128 arithmetic on
    real data and LU on a symmetric matrix must reproduce it,
  * scipy's sparse direct solver (backward error of the supernodal solve),
  * the flop convention (LU = 2 x LLt per task, complex = 4 x real).
"""

import numpy as np
import pytest

from oracle import panel_oracle as O
from oracle import panel_oracle_ext as X
from paper_1405_2636_b200 import flops, sparse
from paper_1405_2636_b200.analysis import AnalyzeOptions, analyze
from paper_1405_2636_b200.errors import NotPositiveDefiniteError, SingularPivotError


def gather(symbol, store):
    """Dense lower (incl. diagonal) from a PanelStore, any dtype."""
    n = symbol.n
    L = np.zeros((n, n), dtype=store.slab.dtype)
    for p in range(symbol.npanels):
        a = store.data[p]
        rm = store.rowmaps[p]
        fc, w = int(symbol.starts[p]), int(symbol.widths[p])
        for c in range(w):
            L[rm[c:], fc + c] = a[c:, c]
    return L


def dense_of(A):
    """Dense matrix of a sparse matrix in either storage."""
    n = A.n
    D = np.zeros((n, n), dtype=A.values.dtype)
    cols = A.entry_cols()
    np.add.at(D, (A.rowidx, cols), A.values)
    if A.stype == sparse.SYMMETRIC_LOWER:
        off = A.rowidx != cols
        np.add.at(D, (cols[off], A.rowidx[off]), A.values[off])
    return D


def rand_general(rng, n, density, cplx=False):
    """Random nonsymmetric, diagonally dominant sparse matrix (general storage)."""
    mask = (rng.random((n, n)) < density) & ~np.eye(n, dtype=bool)
    V = rng.uniform(-1.0, 1.0, (n, n)) * mask
    if cplx:
        V = V + 1j * rng.uniform(-1.0, 1.0, (n, n)) * mask
    V = V + np.diag(np.abs(V).sum(axis=1) + rng.uniform(0.5, 1.5, n))
    r, c = np.nonzero(V)
    return sparse.from_coo(n, r, c, V[r, c], sparse.GENERAL), V


def lu_dense_from(an, store, ustore):
    """(L unit lower, U upper) of P A P^T from the two LU slabs."""
    Lfull = gather(an.symbol, store)
    Ut = gather(an.symbol, ustore)
    d = np.diagonal(Lfull).copy()
    L = np.tril(Lfull, -1) + np.eye(an.symbol.n)
    U = np.tril(Ut, -1).T + np.diag(d)
    return L, U


@pytest.mark.parametrize("cplx", [False, True])
def test_lu_matches_dense_doolittle(cplx):
    rng = np.random.default_rng(7 + cplx)
    for n, dens in ((40, 0.1), (90, 0.05), (150, 0.03)):
        A, _ = rand_general(rng, n, dens, cplx)
        an = analyze(A, AnalyzeOptions(form="lu", nd_leaf=8, split_width=16))
        st, ut = X.factor_analysis(an)
        Ap = dense_of(an.A_perm)
        Ld, Ud = X.dense_lu(Ap)
        L, U = lu_dense_from(an, st, ut)
        assert np.abs(L - Ld).max() <= 1e-12 * np.abs(Ld).max()
        assert np.abs(U - Ud).max() <= 1e-12 * np.abs(Ud).max()


def test_lu_convdiff_solve_vs_scipy():
    import scipy.sparse as sps
    import scipy.sparse.linalg as spla
    for cs in (None, 1.0):
        A = sparse.gen_convdiff27(10, complex_shift=cs)
        an = analyze(A, AnalyzeOptions(form="lu"))
        st, ut = X.factor_analysis(an)
        b = sparse.spmv(A, np.ones(A.n) * (1 + 0.5j if cs else 1.0))
        x = X.solve(an.symbol, st, ut, b, "lu", an.perm.perm)
        D = dense_of(A)
        xs = spla.spsolve(sps.csc_matrix(D), b)
        assert sparse.backward_error(A, x, b) <= 1e-13
        assert np.abs(x - xs).max() <= 1e-10 * np.abs(xs).max()


@pytest.mark.parametrize("form", ["llt", "ldlt"])
def test_complex_symmetric_matches_dense(form):
    rng = np.random.default_rng(11)
    n = 80
    mask = np.tril(rng.random((n, n)) < 0.08, -1)
    V = (rng.uniform(-1, 1, (n, n)) + 1j * rng.uniform(-1, 1, (n, n))) * mask
    Ad = V + V.T  # complex SYMMETRIC (not Hermitian)
    Ad = Ad + np.diag(np.abs(Ad).sum(axis=1) + 1.0 + 0.3j)
    r, c = np.nonzero(np.tril(Ad))
    A = sparse.from_coo(n, r, c, Ad[r, c], sparse.SYMMETRIC_LOWER)
    an = analyze(A, AnalyzeOptions(form=form, nd_leaf=8, split_width=16))
    st, _ = X.factor_analysis(an)
    Ap = dense_of(an.A_perm)
    G = gather(an.symbol, st)
    Ld, dd = X.dense_ldlt(Ap)
    if form == "ldlt":
        L = np.tril(G, -1) + np.eye(n)
        assert np.abs(L - Ld).max() <= 1e-12 * np.abs(Ld).max()
        assert np.abs(np.diagonal(G) - dd).max() <= 1e-12 * np.abs(dd).max()
    else:
        Lc = Ld * np.sqrt(dd)[None, :]  # A = (L D^1/2)(L D^1/2)^T, principal sqrt
        assert np.abs(G - Lc).max() <= 1e-12 * np.abs(Lc).max()
    b = Ap @ np.ones(n)
    x = X.solve(an.symbol, st, None, b, form)
    assert np.linalg.norm(Ap @ x - b) / np.linalg.norm(b) <= 1e-13


@pytest.mark.parametrize("form", ["llt", "ldlt"])
def test_ext_oracle_reproduces_real_oracle(form):
    """Real symmetric input: the extension oracle (real and complex128
    arithmetic) and LU on the same matrix reproduce the pinned real oracle."""
    A = sparse.gen_laplacian(3, (7, 7, 7))
    if form == "ldlt":
        A = sparse.shift_diagonal(A, 0.5)
    an = analyze(A, AnalyzeOptions(form=form))
    ref = O.factor_analysis(an).slab
    st, _ = X.factor_analysis(an)
    assert np.abs(st.slab - ref).max() <= 1e-13 * np.abs(ref).max()
    Ac = sparse.SparseMatrix(A.n, A.colptr, A.rowidx, A.values.astype(np.complex128), A.stype)
    anc = analyze(Ac, AnalyzeOptions(form=form))
    stc, _ = X.factor_analysis(anc)
    assert np.abs(stc.slab.imag).max() == 0.0
    assert np.abs(stc.slab.real - ref).max() <= 1e-13 * np.abs(ref).max()
    if form == "ldlt":  # LU of a symmetric matrix: L equal, U^T = L D
        anl = analyze(A, AnalyzeOptions(form="lu"))
        stl, utl = X.factor_analysis(anl)
        assert np.abs(stl.slab - ref).max() <= 1e-12 * np.abs(ref).max()
        L = gather(anl.symbol, stl)
        d = np.diagonal(L)
        Lu = np.tril(L, -1)
        Ut = np.tril(gather(anl.symbol, utl), -1)
        assert np.abs(Ut - Lu * d[None, :]).max() <= 1e-12 * np.abs(Ut).max()


def test_lu_singular_pivot():
    # zero leading pivot after the ordering: a 2x2 block [[0, 1], [1, 0]] plus a diagonal
    n = 6
    D = np.diag(np.arange(1.0, n + 1))
    D[:2, :2] = [[0.0, 1.0], [2.0, 0.0]]
    r, c = np.nonzero(D)
    A = sparse.from_coo(n, r, c, D[r, c], sparse.GENERAL)
    an = analyze(A, AnalyzeOptions(form="lu", ordering="natural"))
    with pytest.raises(SingularPivotError) as ei:
        X.factor_analysis(an)
    assert ei.value.column == 0


def test_complex_llt_zero_pivot_raises():
    A = sparse.from_coo(2, np.array([0, 1, 1]), np.array([0, 0, 1]),
                        np.array([1.0 + 0j, 1.0 + 0j, 1.0 + 0j]), sparse.SYMMETRIC_LOWER)
    an = analyze(A, AnalyzeOptions(form="llt", ordering="natural"))
    with pytest.raises(NotPositiveDefiniteError) as ei:
        X.factor_analysis(an)
    assert ei.value.column == 1


def test_lu_and_complex_flop_convention():
    A = sparse.gen_convdiff27(8)
    an_l = analyze(A, AnalyzeOptions(form="lu"))
    an_s = analyze(sparse.symmetrize_pattern(A), AnalyzeOptions(form="llt"))
    assert an_l.flops == 2 * an_s.flops
    Ac = sparse.gen_convdiff27(8, complex_shift=1.0)
    an_c = analyze(Ac, AnalyzeOptions(form="lu"))
    assert an_c.flops == 8 * an_s.flops
    assert flops.total_flops(an_s.symbol, "llt", True) == 4 * an_s.flops
