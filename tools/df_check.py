"""Dataflow vs level schedule: parity against the oracle and timing (dev tool).

  python tools/df_check.py [N ...]"""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from oracle import panel_oracle as O
from paper_1405_2636_b200 import sparse
from paper_1405_2636_b200.analysis import analyze, AnalyzeOptions
from paper_1405_2636_b200.pipeline import get_engine, default_pivot_threshold, DeviceStore


def run(eng, an, form, thr, sched, reps=3):
    eng.set_schedule(sched)
    store = eng.new_store()
    best = 1e30
    for _ in range(reps):
        eng.assemble(store, an.A_perm)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); eng.factor(store, form, thr); e1.record()
        eng.check(form)
        best = min(best, e0.elapsed_time(e1))
    return store.cpu().numpy(), best


cases = [("2d", 16, "llt"), ("3d", 8, "llt"), ("3d", 8, "ldlt"), ("3d", 16, "llt"), ("3d", 16, "ldlt"),
         ("3d", 24, "llt")]
sizes = [int(a) for a in sys.argv[1:]]
for dim, N, form in cases + [("3d", n, "llt") for n in sizes]:
    A = sparse.gen_laplacian(2 if dim == "2d" else 3, (N,) * (2 if dim == "2d" else 3))
    if form == "ldlt":
        A = sparse.shift_diagonal(A, 0.5)
    an = analyze(A, AnalyzeOptions(form=form))
    thr = default_pivot_threshold(an.A_perm)
    t = time.time(); eng = get_engine(an); tp = time.time() - t
    di = eng.dataflow_info()
    lv, tl = run(eng, an, form, thr, "level")
    df, td = run(eng, an, form, thr, "dataflow")
    d2, _ = run(eng, an, form, thr, "dataflow", reps=1)
    err_ld = np.abs(lv - df).max() / np.abs(lv).max()
    msg = f"{dim} {N} {form}: plan {tp:.2f}s tasks {di['ntasks']} est {di['est_ms']:.2f} ms | level {tl:.3f} ms dataflow {td:.3f} ms ({an.flops/td/1e9:.1f} TF) | df-vs-level {err_ld:.2e} df bitwise-repeat {np.array_equal(df, d2)}"
    if N <= 24:
        ref = O.factor_analysis(an).slab
        msg += f" | df-vs-oracle {np.abs(df - ref).max() / np.abs(ref).max():.2e}"
    print(msg, flush=True)
    print("   tasks by type", di["tasks_by_type"], flush=True)
