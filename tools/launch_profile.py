"""Per-launch device time of one factorization (non-graph, CUDA events).

Writes gpurun_out/launches_<N>.csv (launch, kind, level, items, ms) and
prints a summary by kind and the most expensive launches."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1405_2636_b200 import sparse
from paper_1405_2636_b200.analysis import analyze, AnalyzeOptions
from paper_1405_2636_b200.pipeline import get_engine, default_pivot_threshold

N = int(sys.argv[1]) if len(sys.argv) > 1 else 60
form = sys.argv[2] if len(sys.argv) > 2 else "llt"
A = sparse.gen_laplacian(3, (N, N, N))
if form == "ldlt":
    A = sparse.shift_diagonal(A, 0.5)
an = analyze(A, AnalyzeOptions(form=form))
eng = get_engine(an)
thr = default_pivot_threshold(an.A_perm)
store = eng.new_store()
for _ in range(2):
    eng.assemble(store, an.A_perm); eng.factor(store, form, thr); eng.check(form)
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
eng.assemble(store, an.A_perm)
e0.record(); eng.factor(store, form, thr); e1.record(); eng.check(form)
graph_ms = e0.elapsed_time(e1)
eng.assemble(store, an.A_perm)
tb = eng.factor_timed(store, form, thr, per_launch=True)
kind, lvl, cnt, br = eng.launch_table(branches=True)
ms = tb["per_launch_ms"]
fl, by = eng.launch_work()
os.makedirs("gpurun_out", exist_ok=True)
with open(f"gpurun_out/launches_{N}_{form}.csv", "w") as fh:
    fh.write("launch,kind,level,items,branch,ms,flops,bytes\n")
    for i in range(len(ms)):
        fh.write(f"{i},{eng.KIND_NAMES[kind[i]]},{lvl[i]},{cnt[i]},{br[i]},{ms[i]:.5f},{fl[i]:.6g},{by[i]:.6g}\n")
print(f"branches: {int(br.max())} groups; top launches {int((br == 0).sum())} of {len(br)}")
print(f"N={N} graph {graph_ms:.3f} ms ({an.flops/graph_ms/1e9:.2f} TFlop/s); non-graph sum {ms.sum():.3f} ms, launches {len(ms)}")
for k in range(len(eng.KIND_NAMES)):
    sel = kind == k
    if sel.any():
        print(f"  {eng.KIND_NAMES[k]:18s} launches {sel.sum():5d} items {cnt[sel].sum():9d} ms {ms[sel].sum():8.3f}  mean {ms[sel].mean()*1e3:7.1f} us")
order = np.argsort(-ms)[:15]
for i in order[:12]:
    print(f"  top: launch {i} {eng.KIND_NAMES[kind[i]]} level {lvl[i]} items {cnt[i]} {ms[i]:.3f} ms")
