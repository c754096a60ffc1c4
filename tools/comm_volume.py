"""Communication volume of the multi-GPU factorization (host-only, no GPU).

    python tools/comm_volume.py N G [G ...]

For the subtree partition (distributed.partition) and top ownership
(distributed.top_owners) of the 3D 7-point Laplacian N^3, per top level:

  fan-in   dense : the whole top region all-reduced (ring: 2 (G-1)/G of it
                   sent per rank; total over ranks 2 (G-1) x region)
           exact : every top panel q pulled by its owner from each OTHER rank
                   that contributes to it (a couple p -> q with p in that
                   rank's subtrees, or A's values on rank 0) - P2P reads
  panels   bcast : each top panel sent to all G-1 other ranks
           target: each top panel sent only to the owners of its
                   destinations (other than its own owner) - P2P reads
Bytes in GB (8-byte entries).
"""
import sys

import numpy as np

sys.path.insert(0, __import__("os").path.dirname(__file__) + "/..")
from paper_1405_2636_b200 import sparse  # noqa: E402
from paper_1405_2636_b200.analysis import analyze  # noqa: E402
from paper_1405_2636_b200.distributed import (panel_levels, partition,  # noqa: E402
                                              top_owners)


def volumes(an, G):
    sym = an.symbol
    group = partition(sym, G)
    owner = top_owners(sym, group, G)
    size = (sym.widths * sym.nrows_arr).astype(np.float64) * 8
    top = group < 0
    src = np.repeat(np.arange(sym.npanels), np.diff(sym.blkptr))
    dst = sym.blk_facing
    lev = panel_levels(sym)
    # contributors of every top panel (fan-in from the subtrees)
    sel = top[dst] & ~top[src]
    contrib = {}
    for g, q in set(zip(group[src[sel]].tolist(), dst[sel].tolist())):
        contrib.setdefault(q, set()).add(g)
    # destinations' owners of every top panel (top -> top couples)
    sel = top[src] & top[dst]
    readers = {}
    for p, q in set(zip(src[sel].tolist(), dst[sel].tolist())):
        readers.setdefault(p, set()).add(int(owner[q]))
    tops = np.flatnonzero(top)
    region = size[tops].sum()
    rows = {}
    exact = bcast = target = 0.0
    for q in tops.tolist():
        L = int(lev[q])
        r = rows.setdefault(L, [0, 0.0, 0.0, 0.0, 0.0])
        r[0] += 1
        r[1] += size[q]
        c = set(contrib.get(q, set())) | {0}
        e = len(c - {int(owner[q])}) * size[q]
        b = (G - 1) * size[q]
        t = len(readers.get(q, set()) - {int(owner[q])}) * size[q]
        r[2] += e
        r[3] += b
        r[4] += t
        exact += e
        bcast += b
        target += t
    return group, region, exact, bcast, target, rows


def main(N, Gs):
    an = analyze(sparse.gen_laplacian(3, (N, N, N)))
    sym = an.symbol
    slab = float((sym.widths * sym.nrows_arr).sum()) * 8
    print(f"N={N}: slab {slab / 1e9:.2f} GB, {sym.npanels} panels")
    for G in Gs:
        group, region, exact, bcast, target, rows = volumes(an, G)
        ntop = int((group < 0).sum())
        print(f"\nG={G}: top panels {ntop}, top region {region / 1e9:.3f} GB "
              f"({region / slab:.1%} of the slab)")
        print(f"  fan-in : dense all-reduce {2 * (G - 1) * region / 1e9:.3f} GB total "
              f"(ring), exact P2P pulls {exact / 1e9:.3f} GB")
        print(f"  panels : broadcast to all {bcast / 1e9:.3f} GB, to destination owners only "
              f"{target / 1e9:.3f} GB")
        print(f"  {'level':>5s} {'panels':>6s} {'GB':>8s} {'fanin GB':>9s} {'bcast GB':>9s} {'target GB':>9s}")
        for L in sorted(rows):
            n, s, e, b, t = rows[L]
            print(f"  {L:5d} {n:6d} {s / 1e9:8.3f} {e / 1e9:9.3f} {b / 1e9:9.3f} {t / 1e9:9.3f}")


if __name__ == "__main__":
    main(int(sys.argv[1]), [int(g) for g in sys.argv[2:]] or [2, 4, 8])
