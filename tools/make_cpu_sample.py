"""Stratified CPU-baseline sample of a symbol (for bench.py's cpu_baseline
and --impl reference legs, which then need neither the analysis nor any of
this repository's native libraries).

    python tools/make_cpu_sample.py 120 llt      -> bench_data/cpu_sample_120_llt.npz

Source panels are grouped by width class (STRATA); a task unit = the factor
task of one panel plus every update task it sources (kernels.py:208-309).
From each class, units are drawn uniformly at random (seed 0) among those
costing <= CAP flops until the class's share of the sample budget (or MAXU
units) is reached.  The file holds the drawn panels' block structure and the row maps
of their destinations (global row numbers), plus every class's total flops,
so the CPU rate can be extrapolated per class:
    T_est = sum_s F_s / rate_s,  GFlop/s = total_flops / T_est.
"""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

STRATA = (1, 2, 9, 33, 129, 513, 1 << 30)  # width classes [lo, hi)
BUDGET = 40e9   # sampled flops (about 15 s of one core at the reference's rate)
CAP = 4e9       # no single unit above this (bounded sample; wider units extrapolated)
MAXU = 3000     # units per class (narrow classes: per-task overhead, not flops, is the cost)


def main(size, form):
    from paper_1405_2636_b200 import sparse
    from paper_1405_2636_b200.analysis import AnalyzeOptions, analyze
    from paper_1405_2636_b200.flops import block_flops_array, factor_flops_array
    A = sparse.gen_laplacian(3, (size, size, size))
    if form == "ldlt":
        A = sparse.shift_diagonal(A, 0.5)
    an = analyze(A, AnalyzeOptions(form=form))
    s = an.symbol
    unit = factor_flops_array(s, form).astype(np.float64)
    bf = block_flops_array(s, form).astype(np.float64)
    owner = np.repeat(np.arange(s.npanels), np.diff(s.blkptr))
    np.add.at(unit, owner, bf)
    w = s.widths
    cls = np.searchsorted(np.array(STRATA), w, side="right") - 1
    total = float(unit.sum())
    rng = np.random.default_rng(0)
    pick = []
    F = np.zeros(len(STRATA) - 1)
    for c in range(len(STRATA) - 1):
        members = np.flatnonzero(cls == c)
        F[c] = unit[members].sum()
        if not len(members):
            continue
        share = max(0.03 * BUDGET, BUDGET * F[c] / total)
        cand = members[unit[members] <= CAP]
        if not len(cand):
            cand = members[np.argsort(unit[members])[:1]]
        got = 0.0
        npick0 = len(pick)
        for p in rng.permutation(cand):
            pick.append(int(p))
            got += unit[p]
            if got >= share or len(pick) - npick0 >= MAXU:
                break
    pick = sorted(pick)
    # mini symbol: sampled sources, then their destinations
    dests = sorted({int(q) for p in pick for q in s.blk_facing[s.blkptr[p]:s.blkptr[p + 1]]})
    mini = pick + [q for q in dests if q not in set(pick)]
    mid = {p: i for i, p in enumerate(mini)}
    fc = np.array([s.starts[p] for p in mini], dtype=np.int64)
    pw = np.array([w[p] for p in mini], dtype=np.int64)
    rptr = np.zeros(len(mini) + 1, dtype=np.int64)
    for i, p in enumerate(mini):
        rptr[i + 1] = rptr[i] + (s.rowptr[p + 1] - s.rowptr[p])
    rows = np.concatenate([s.rowdata[s.rowptr[p]:s.rowptr[p + 1]] for p in mini]).astype(np.int64)
    bptr = np.zeros(len(pick) + 1, dtype=np.int64)
    bfr, blr, bfa, blo = [], [], [], []
    for i, p in enumerate(pick):
        b0, b1 = s.blkptr[p], s.blkptr[p + 1]
        bptr[i + 1] = bptr[i] + (b1 - b0)
        bfr += s.blk_fr[b0:b1].tolist()
        blr += s.blk_lr[b0:b1].tolist()
        bfa += [mid[int(q)] for q in s.blk_facing[b0:b1]]
        blo += s.blk_loc[b0:b1].tolist()
    out = os.path.join(ROOT, "bench_data", f"cpu_sample_{size}_{form}.npz")
    np.savez_compressed(out, fc=fc, w=pw, rowptr=rptr, rows=rows, nsrc=len(pick),
                        src_class=cls[pick], src_flops=unit[pick], blkptr=bptr,
                        blk_fr=np.array(bfr, dtype=np.int64), blk_lr=np.array(blr, dtype=np.int64),
                        blk_facing=np.array(bfa, dtype=np.int64),
                        blk_loc=np.array(blo, dtype=np.int64), strata=np.array(STRATA),
                        class_flops=F, class_units=np.bincount(cls, minlength=len(F)),
                        total_flops=total, flops_exact=int(an.flops), form=form, size=size)
    print(out, len(pick), "sources", len(mini), "panels", unit[pick].sum() / 1e9, "GFlop sampled",
          os.path.getsize(out) / 1e6, "MB")


if __name__ == "__main__":
    main(int(sys.argv[1]), sys.argv[2] if len(sys.argv) > 2 else "llt")
