"""CPU ORACLE for LU and complex factorizations - TEST INFRASTRUCTURE ONLY.

The reference package factors only real LLt / LDLt (kernels.py:19-22) and
symmetrizes nonsymmetric input (sparse.py:201-229).  The north star asks for
LLt / LDLt / LU in real and complex double; this module restates the paper's
nonsymmetric variant (the symbolic structure of A + A^T,
"the factorization steps 2 and 3 are duplicated for the L and U factors",
static pivoting) on the reference's own data structures, mirroring
kernels.py:208-309 operation for operation:

Storage (the PanelStore layout twice, symbolic.py:318-335): `a` holds L
(strict lower; unit diagonal implicit) with U's diagonal on the diagonal;
`u` holds U transposed: u[r, j] = U[fc + j, row r] for every local row r
below j (diagonal-block strict lower part and the off-diagonal rows).  For
the symmetric forms U^T = L (LLt) / L D (LDLt), so `u` is not stored.

* panel factorization, left-looking column sweep over the whole tall panel
  (the LU restatement of kernels.py:208-247):
      s = a[j:, j] - a[j:, :j] @ u[j, :j];  piv = s[0]
      |piv| <= thr -> SingularPivotError(fc + j, piv)
      a[j, j] = piv;  a[j+1:, j] = s[1:] / piv
      u[j+1:, j] -= u[j+1:, :j] @ a[j, :j]
* couple update (sparse_gemm with direct scatter, kernels.py:128-136 twice):
      L: dst_a[dloc[c:], col0 + c]   -= a[loc + c:, :]     @ u[loc + c, :]
      U: dst_u[dloc[c+1:], col0 + c] -= u[loc + c + 1:, :] @ a[loc + c, :]
* complex: the same sweeps in complex arithmetic (symmetric forms are
  complex-symmetric A = L L^T / L D L^T, no conjugation); the pivot test is
  |piv| <= thr for every complex form (real LLt keeps piv <= thr).
* solve: L y = b (forward, unit for LDLt / LU), diagonal scaling (LDLt),
  U x = y (backward; U = L^T for LLt, L^T for LDLt, from `u` for LU).

Pinned by tests/test_oracle_ext.py against dense no-pivot LU / LDLt /
Cholesky written directly in numpy, and against scipy's sparse solver.
"""

from __future__ import annotations

import numpy as np

from paper_1405_2636_b200.errors import (NotPositiveDefiniteError, SingularPivotError,
                                         StructuralError)

LLT, LDLT, LU = "llt", "ldlt", "lu"


def _fails(piv, thr, form):
    if form == LLT and not np.iscomplexobj(piv):
        return piv <= thr
    return abs(piv) <= thr


def _raise(form, col, piv):
    if form == LLT:
        raise NotPositiveDefiniteError(col, piv)
    raise SingularPivotError(col, piv)


def factor_panel(a, u, fc, form, thr):
    """In-place factor of one panel (a: L part, u: U^T part for LU)."""
    w = a.shape[1]
    d = np.empty(w, dtype=a.dtype)
    for j in range(w):
        if form == LU:
            s = a[j:, j] - a[j:, :j] @ u[j, :j]
        elif form == LDLT:
            s = a[j:, j] - a[j:, :j] @ (d[:j] * a[j, :j])
        else:
            s = a[j:, j] - a[j:, :j] @ a[j, :j]
        piv = s[0]
        if _fails(piv, thr, form):
            _raise(form, fc + j, piv)
        if form == LLT:
            r = np.sqrt(piv)
            a[j, j] = r
            a[j + 1:, j] = s[1:] / r
        else:
            d[j] = piv
            a[j, j] = piv
            a[j + 1:, j] = s[1:] / piv
            if form == LU:
                u[j + 1:, j] -= u[j + 1:, :j] @ a[j, :j]


def couples_of(symbol, p):
    b0, b1 = int(symbol.blkptr[p]), int(symbol.blkptr[p + 1])
    out = {}
    for b in range(b0, b1):
        out.setdefault(int(symbol.blk_facing[b]), []).append(b)
    return dict(sorted(out.items()))


def update_couple(symbol, store, ustore, p, q, blocks, form):
    """All blocks of p facing q, scattered directly into q (both factors for LU)."""
    if not blocks:
        raise StructuralError(f"no blocks of panel {p} face panel {q}")
    a, dst = store.data[p], store.data[q]
    u = ustore.data[p] if form == LU else None
    du = ustore.data[q] if form == LU else None
    w = int(symbol.widths[p])
    rm, qrm = store.rowmaps[p], store.rowmaps[q]
    qfc = int(symbol.starts[q])
    dsc = np.diagonal(a[:w, :w]).copy() if form == LDLT else None
    loc0 = int(symbol.blk_loc[blocks[0]])
    full = np.searchsorted(qrm, rm[loc0:])
    for b in blocks:
        loc = int(symbol.blk_loc[b])
        h = int(symbol.blk_lr[b] - symbol.blk_fr[b])
        col0 = int(symbol.blk_fr[b]) - qfc
        dloc = full[loc - loc0:]
        for c in range(h):
            if form == LU:
                dst[dloc[c:], col0 + c] -= a[loc + c:, :] @ u[loc + c, :]
                du[dloc[c + 1:], col0 + c] -= u[loc + c + 1:, :] @ a[loc + c, :]
            else:
                row = a[loc + c, :] if dsc is None else dsc * a[loc + c, :]
                dst[dloc[c:], col0 + c] -= a[loc + c:, :] @ row


def factorize(symbol, store, ustore, form, thr):
    """Canonical order (kernels.py:318-326): ascending p, then ascending q."""
    for p in range(symbol.npanels):
        factor_panel(store.data[p], ustore.data[p] if form == LU else None,
                     int(symbol.starts[p]), form, thr)
        for q, blocks in couples_of(symbol, p).items():
            update_couple(symbol, store, ustore, p, q, blocks, form)


def solve(symbol, store, ustore, b, form, perm=None):
    """x with A x = b (the contract of kernels.py:332-382, all forms)."""
    n = symbol.n
    dt = np.result_type(store.slab.dtype, np.asarray(b).dtype)
    if perm is None:
        perm = np.arange(n, dtype=np.int64)
    x = np.empty(n, dtype=dt)
    x[perm] = b
    unit = form != LLT
    for p in range(symbol.npanels):
        a = store.data[p]
        fc, lc = int(symbol.starts[p]), int(symbol.starts[p + 1])
        w = lc - fc
        rows = symbol.panel_rows(p)
        y = x[fc:lc]
        for j in range(w):
            if not unit:
                y[j] /= a[j, j]
            y[j + 1:] -= a[j + 1:w, j] * y[j]
        if len(rows):
            x[rows] -= a[w:, :] @ y
    for p in range(symbol.npanels):  # D (LDLt) / U's diagonal (LU)
        if form in (LDLT, LU):
            fc, lc = int(symbol.starts[p]), int(symbol.starts[p + 1])
            x[fc:lc] /= np.diagonal(store.data[p][:lc - fc, :lc - fc])
    for p in range(symbol.npanels - 1, -1, -1):
        a = store.data[p]
        t = ustore.data[p] if form == LU else a
        fc, lc = int(symbol.starts[p]), int(symbol.starts[p + 1])
        w = lc - fc
        rows = symbol.panel_rows(p)
        y = x[fc:lc]
        if len(rows):
            if form == LU:
                # U[j, r] = t[r, j]; U = D_U * (unit upper): scale by 1 / U_jj
                y -= (t[w:, :].T @ x[rows]) / np.diagonal(a[:w, :w])
            else:
                y -= t[w:, :].T @ x[rows]
        for j in range(w - 1, -1, -1):
            if form == LU:
                y[j] -= (t[j + 1:w, j] @ y[j + 1:w]) / a[j, j]
            else:
                y[j] -= t[j + 1:w, j] @ y[j + 1:w]
                if not unit:
                    y[j] /= a[j, j]
    return x[perm]


def allocate(symbol, A, form):
    """(store, ustore) with A's entries scattered in (allocate_panels,
    symbolic.py:338-350, extended: upper entries of a general A go to u at
    the transposed position)."""
    from paper_1405_2636_b200.symbolic import PanelStore, assembly_positions_any
    dt = np.result_type(A.values.dtype, np.float64)
    store = PanelStore(symbol, dtype=dt)
    ustore = PanelStore(symbol, dtype=dt) if form == LU else None
    cols = A.entry_cols()
    rows = A.rowidx
    low = rows >= cols
    store.slab[assembly_positions_any(symbol, rows[low], cols[low])] = A.values[low]
    if form == LU and (~low).any():
        ustore.slab[assembly_positions_any(symbol, cols[~low], rows[~low])] = A.values[~low]
    return store, ustore


def pivot_threshold(A):
    cols = A.entry_cols()
    on = A.rowidx == cols
    return 1e-13 * float(np.abs(A.values[on]).max()) if on.any() else 0.0


def factor_analysis(an, form=None):
    form = form or an.options.form
    store, ustore = allocate(an.symbol, an.A_perm, form)
    factorize(an.symbol, store, ustore, form, pivot_threshold(an.A_perm))
    return store, ustore


# ---------------------------------------------------------------------------
# dense references (pin the restatement)

def dense_lu(Ad):
    """No-pivot Doolittle LU: (L unit lower, U upper)."""
    A = np.array(Ad, dtype=np.result_type(Ad, np.float64))
    n = A.shape[0]
    for k in range(n):
        A[k + 1:, k] /= A[k, k]
        A[k + 1:, k + 1:] -= np.outer(A[k + 1:, k], A[k, k + 1:])
    L = np.tril(A, -1) + np.eye(n)
    return L, np.triu(A)


def dense_ldlt(Ad):
    """No-pivot LDL^T (complex symmetric allowed): (L unit lower, d)."""
    L, U = dense_lu(Ad)
    return L, np.diagonal(U).copy()
