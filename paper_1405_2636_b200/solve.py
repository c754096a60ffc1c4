"""Supernodal triangular solve over a factored panel store (host).

Contract of the reference's `supernodal_solve` (kernels.py:332-382):
permute, forward substitution per panel ascending (unit-lower + divide by d
for LDLt), backward substitution descending, un-permute.  Dense diagonal
blocks use LAPACK triangular solves (scipy).  FactorResult.solve runs the
GPU solve (ps_solve, csrc/ps_solve.cuh) on a device-resident factor; this
host path serves a factor that only exists on the host (a FactorResult
rebuilt from a downloaded store) and the host residual checks.
"""

from __future__ import annotations

import numpy as np
from scipy.linalg import solve_triangular

from .errors import DivergentSolveError

LDLT = "ldlt"


def supernodal_solve(symbol, store, b, form="llt", perm=None):
    n = symbol.n
    b = np.asarray(b, dtype=np.float64)
    if b.shape != (n,):
        raise ValueError("right-hand side length mismatch")
    if perm is None:
        perm = np.arange(n, dtype=np.int64)
    x = np.empty(n)
    x[perm] = b
    starts = symbol.starts
    ldlt = form == LDLT
    for p in range(symbol.npanels):
        a = store.data[p]
        fc, lc = int(starts[p]), int(starts[p + 1])
        w = lc - fc
        rows = symbol.panel_rows(p)
        if w == 1:
            if not ldlt:
                x[fc] /= a[0, 0]
        else:
            x[fc:lc] = solve_triangular(a[:w, :w], x[fc:lc], lower=True,
                                        unit_diagonal=ldlt, check_finite=False)
        if len(rows):
            x[rows] -= a[w:, :] @ x[fc:lc]
        if ldlt:
            d = np.diagonal(a[:w, :w])
            if np.any(d == 0.0):
                raise DivergentSolveError("zero LDLt diagonal in solve")
            x[fc:lc] /= d
    for p in range(symbol.npanels - 1, -1, -1):
        a = store.data[p]
        fc, lc = int(starts[p]), int(starts[p + 1])
        w = lc - fc
        rows = symbol.panel_rows(p)
        if len(rows):
            x[fc:lc] -= a[w:, :].T @ x[rows]
        if w == 1:
            if not ldlt:
                x[fc] /= a[0, 0]
        else:
            x[fc:lc] = solve_triangular(a[:w, :w], x[fc:lc], lower=True, trans="T",
                                        unit_diagonal=ldlt, check_finite=False)
    return x[perm]
