"""Issued DMMA work vs the metric's flops for the inter-panel update tiles.

Mirrors the plan's tiling (ps_b200.cu emit_tiles: couple (p -> q) covers
source rows [loc0, nrows) x facing rows [loc0, loc0 + N), tm x tn tiles,
tiles entirely above the diagonal skipped; K padded to the pipeline chunk)
on the host symbol, so shapes can be compared without a GPU:

    python tools/tile_waste.py 60 [tm tn kc]
"""
import sys

import numpy as np

sys.path.insert(0, __import__("os").path.dirname(__file__) + "/..")
from paper_1405_2636_b200 import sparse  # noqa: E402
from paper_1405_2636_b200.analysis import analyze  # noqa: E402


def couples(sym):
    bp = sym.blkptr
    fac = sym.blk_facing
    for p in range(sym.npanels):
        b0, b1 = bp[p], bp[p + 1]
        if b1 == b0:
            continue
        f = fac[b0:b1]
        cut = np.flatnonzero(np.diff(f)) + 1
        starts = np.concatenate([[0], cut])
        ends = np.concatenate([cut, [b1 - b0]])
        for s, e in zip(starts, ends):
            yield p, b0 + s, b0 + e


def main(N, tm=64, tn=64, kc=16, small_w=8, shapes=0):
    """shapes=1: each tile issues the smallest of 64|32 rows x 64|32 columns
    holding it (the kernels' tile_shape); shapes=8: ceil8(ni) x ceil8(nj)."""
    an = analyze(sparse.gen_laplacian(3, (N, N, N)))
    sym = an.symbol
    w = sym.widths
    nr = sym.nrows_arr
    metric = issued = useful = 0.0
    hist = {}
    for p, g0, g1 in couples(sym):
        K = int(w[p])
        if K <= small_w:
            continue
        loc = sym.blk_loc[g0:g1]
        h = sym.blk_lr[g0:g1] - sym.blk_fr[g0:g1]
        m = nr[p] - loc
        metric += float((2 * m * h * K).sum())
        loc0 = int(loc[0])
        Nf = int(h.sum())
        kpad = -(-K // kc) * kc
        for j in range(loc0, loc0 + Nf, tn):
            nj = min(tn, loc0 + Nf - j)
            for i in range(loc0, int(nr[p]), tm):
                ni = min(tm, int(nr[p]) - i)
                if i + ni - 1 < j:
                    continue
                if shapes == 1:
                    issued += 2.0 * (32 if ni <= 32 else 64) * (32 if nj <= 32 else 64) * kpad
                elif shapes == 2:
                    issued += 2.0 * (32 if ni <= 32 else 64) * (-(-nj // 8) * 8) * kpad
                elif shapes == 16:
                    issued += 2.0 * (-(-ni // 16) * 16) * (-(-nj // 16) * 16) * kpad
                elif shapes == 8:
                    issued += 2.0 * (-(-ni // 8) * 8) * (-(-nj // 8) * 8) * kpad
                else:
                    issued += 2.0 * tm * tn * kpad
                # entries on/below the diagonal of the destination (i >= j)
                ii = np.arange(i, i + ni)[:, None]
                jj = np.arange(j, j + nj)[None, :]
                useful += 2.0 * K * float((ii >= jj).sum())
                key = (ni == tm, nj == tn)
                hist[key] = hist.get(key, 0) + 1
    print(f"N={N} tile {tm}x{tn} kc={kc}: metric {metric:.4e}  useful(lower) {useful:.4e}  "
          f"issued {issued:.4e}  metric/issued {metric / issued:.3f}  useful/issued {useful / issued:.3f}")
    print("tiles (full rows, full cols):", hist)


if __name__ == "__main__":
    a = [int(x) for x in sys.argv[1:]]
    main(*a)
