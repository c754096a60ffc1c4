"""Flop accounting - the metric's numerator.

Same cost model as the reference (`kernels.py:142-179`): potrf(k) =
k(k+1)(2k+1)/6, trsm(m,k) = m k^2, gemm = 2 m n k per block with
m = nrows - loc (full h x h head square), plus w^2 + m w per factor and
m w per block for LDLt.  Vectorized over the array symbol.

LU (no reference counterpart; PaStiX convention, "steps 2
and 3 are duplicated for the L and U factors"): twice the LLt count of every
task - getrf(k) = 2 potrf(k), two TRSMs, two scatter GEMMs.  Complex
arithmetic counts 4 real flops per complex multiply-add slot (x4).
"""

from __future__ import annotations

import numpy as np

LLT = "llt"
LDLT = "ldlt"
LU = "lu"


def flops_potrf(k):
    return k * (k + 1) * (2 * k + 1) // 6


def flops_trsm(m, k):
    return m * k * k


def flops_gemm(m, n, k):
    return 2 * m * n * k


def factor_task_flops(panel, form=LLT):
    w = panel.width
    m = len(panel.rows)
    f = flops_potrf(w) + flops_trsm(m, w)
    if form == LDLT:
        f += w * w + m * w
    if form == LU:
        f *= 2
    return f


def update_task_flops(panel, blocks, form=LLT):
    w = panel.width
    tot = 0
    for b in blocks:
        m = panel.nrows - b.loc
        tot += flops_gemm(m, b.height, w)
        if form == LDLT:
            tot += m * w
    return 2 * tot if form == LU else tot


def factor_flops_array(symbol, form=LLT):
    """Per-panel factor-task flops (int64 array)."""
    w = symbol.widths.astype(np.int64)
    m = np.diff(symbol.rowptr).astype(np.int64)
    f = w * (w + 1) * (2 * w + 1) // 6 + m * w * w
    if form == LDLT:
        f = f + w * w + m * w
    return 2 * f if form == LU else f


def block_flops_array(symbol, form=LLT):
    """Per-block update flops (int64 array, aligned with blk_*)."""
    nb = symbol.block_count()
    owner = np.repeat(np.arange(symbol.npanels, dtype=np.int64), np.diff(symbol.blkptr))
    w = symbol.widths[owner].astype(np.int64)
    m = symbol.nrows_arr[owner] - symbol.blk_loc
    h = symbol.blk_lr - symbol.blk_fr
    f = 2 * m * h * w
    if form == LDLT:
        f = f + m * w
    assert len(f) == nb
    return 2 * f if form == LU else f


def total_flops(symbol, form=LLT, complex_=False):
    f = int(factor_flops_array(symbol, form).sum() + block_flops_array(symbol, form).sum())
    return 4 * f if complex_ else f
