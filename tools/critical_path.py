"""Critical path of the factorization graph from per-launch device times.

    python tools/critical_path.py N [form]      (GPU: times one non-graph pass)
    python tools/critical_path.py --csv gpurun_out/launches_N_form.csv  (offline)

Replays the launch list with the graph's branch semantics (ps_b200.cu
enqueue_range: forks, cross-waits and joins between the main stream and the
side branches) and every launch's isolated duration, assuming no slowdown
from branches sharing the GPU.  Prints the makespan (a lower bound of the
graph time) and the critical path's time by kernel kind and level band.
"""
import csv
import sys
from collections import defaultdict

import numpy as np

MARK = {"join": 9, "fork": 10, "xwait": 11}


def simulate(kind, count, branch, ms):
    ready = defaultdict(float)      # stream -> time its last work ends
    pred = defaultdict(lambda: -1)  # stream -> last launch on it (critical chain)
    started = set()
    start = np.zeros(len(kind))
    end = np.zeros(len(kind))
    cp_prev = np.full(len(kind), -1)
    for i, (k, c, b, d) in enumerate(zip(kind, count, branch, ms)):
        if k == "fork":
            if ready[0] >= ready[b]:
                ready[b], pred[b] = ready[0], pred[0]
            started.add(b)
            continue
        if k == "xwait":  # branch c waits for branch b (0: the main stream)
            if (b == 0 or b in started) and ready[b] > ready[c]:
                ready[c], pred[c] = ready[b], pred[b]
            if c and (b == 0 or b in started):
                started.add(c)
            continue
        if k == "join":
            if b in started:
                if ready[b] > ready[0]:
                    ready[0], pred[0] = ready[b], pred[b]
                if c:
                    started.discard(b)
            continue
        if b > 0 and b not in started:
            if ready[0] >= ready[b]:
                ready[b], pred[b] = ready[0], pred[0]
            started.add(b)
        start[i] = ready[b]
        end[i] = start[i] + d
        cp_prev[i] = pred[b]
        ready[b], pred[b] = end[i], i
    last = int(np.argmax(end))
    chain = []
    while last >= 0:
        chain.append(last)
        last = int(cp_prev[last])
    return float(end.max()), chain[::-1]


def report(rows):
    kind = [r["kind"] for r in rows]
    ms = np.array([float(r["ms"]) for r in rows])
    lv = np.array([int(r["level"]) for r in rows])
    cnt = [int(r["items"]) for r in rows]
    br = [int(r["branch"]) for r in rows]
    mk, chain = simulate(kind, cnt, br, ms)
    print(f"launches {len(rows)}, serialized {ms.sum():.2f} ms, simulated makespan {mk:.2f} ms, "
          f"critical path {len(chain)} launches")
    by = defaultdict(float)
    for i in chain:
        by[kind[i]] += ms[i]
    for k, v in sorted(by.items(), key=lambda x: -x[1]):
        print(f"  {k:18s} {v:8.2f} ms on the critical path (of {ms[[j for j in range(len(kind)) if kind[j] == k]].sum():8.2f})")
    bands = defaultdict(float)
    for i in chain:
        L = lv[i]
        bands[(L // 20) * 20] += ms[i]
    print("  by level band:", ", ".join(f"{b}-{b + 19}: {v:.1f}" for b, v in sorted(bands.items())))
    return mk, chain


if __name__ == "__main__":
    if sys.argv[1] == "--csv":
        rows = list(csv.DictReader(open(sys.argv[2])))
        report(rows)
        sys.exit(0)
    import torch  # noqa: F401
    sys.path.insert(0, ".")
    from paper_1405_2636_b200 import sparse
    from paper_1405_2636_b200.analysis import AnalyzeOptions, analyze
    from paper_1405_2636_b200.pipeline import default_pivot_threshold, get_engine
    N = int(sys.argv[1])
    form = sys.argv[2] if len(sys.argv) > 2 else "llt"
    cplx = form == "luc"  # complex LU
    if cplx:
        form = "lu"
    A = (sparse.gen_convdiff27(N, complex_shift=1.0 if cplx else None) if form == "lu"
         else sparse.gen_laplacian(3, (N, N, N)))
    if form == "ldlt":
        A = sparse.shift_diagonal(A, 0.5)
    an = analyze(A, AnalyzeOptions(form=form))
    eng = get_engine(an)
    thr = default_pivot_threshold(an.A_perm)
    store = eng.new_store(form, an.is_complex)
    for _ in range(2):
        eng.assemble(store, an.A_perm, form=form)
        eng.factor(store, form, thr)
    eng.check(form)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    eng.assemble(store, an.A_perm, form=form)
    e0.record()
    eng.factor(store, form, thr)
    e1.record()
    eng.check(form)
    print(f"graph {e0.elapsed_time(e1):.2f} ms")
    eng.assemble(store, an.A_perm, form=form)
    tb = eng.factor_timed(store, form, thr, per_launch=True)
    k, lv, cnt, br = eng.launch_table(branches=True)
    rows = [{"kind": eng.KIND_NAMES[k[i]], "level": lv[i], "items": cnt[i], "branch": br[i],
             "ms": tb["per_launch_ms"][i]} for i in range(len(k))]
    report(rows)
