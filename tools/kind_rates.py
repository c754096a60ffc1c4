"""Per launch kind: time, flops (tile convention) and rate, one non-graph
factorization (dev tool).  python tools/kind_rates.py [N] [form]"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1405_2636_b200 import sparse
from paper_1405_2636_b200.analysis import analyze, AnalyzeOptions
from paper_1405_2636_b200.pipeline import get_engine, default_pivot_threshold
N = int(sys.argv[1]) if len(sys.argv) > 1 else 60
form = sys.argv[2] if len(sys.argv) > 2 else "llt"
cplx = len(sys.argv) > 3 and sys.argv[3] == "complex"
A = (sparse.gen_convdiff27(N, complex_shift=1.0 if cplx else None) if form == "lu"
     else sparse.gen_laplacian(3, (N, N, N)))
if form == "ldlt":
    A = sparse.shift_diagonal(A, 0.5)
an = analyze(A, AnalyzeOptions(form=form))
eng = get_engine(an)
thr = default_pivot_threshold(an.A_perm)
store = eng.new_store(form, an.is_complex)
eng.assemble(store, an.A_perm, form=form); eng.factor(store, form, thr); eng.check(form)
eng.assemble(store, an.A_perm, form=form)
tb = eng.factor_timed(store, form, thr, per_launch=True)
eng.check(form)
kinds, lv, cnt = eng.launch_table()
fl, by = eng.launch_work()
ms = tb["per_launch_ms"]
print(f"N={N} {form}: launches {len(ms)} sum {ms.sum():.2f} ms")
for k, name in enumerate(eng.KIND_NAMES):
    sel = kinds == k
    if sel.any() and ms[sel].sum() > 0:
        print(f"  {name:20s} n {sel.sum():5d} ms {ms[sel].sum():9.2f} flops {fl[sel].sum():.3e} "
              f"rate {fl[sel].sum()/ms[sel].sum()/1e9:7.2f} TF/s  bytes/time {by[sel].sum()/ms[sel].sum()/1e6:7.1f} GB/s")
sel = kinds == 3
big = sel & (fl > np.quantile(fl[sel], 0.9))
print(f"  k_update inter-panel: top-10% launches by flops: {big.sum()} launches, {ms[big].sum():.1f} ms, "
      f"{fl[big].sum()/ms[big].sum()/1e9:.2f} TF/s")
order = np.argsort(-ms)[:10]
for i in order:
    print(f"   launch {i} {eng.KIND_NAMES[kinds[i]]} level {lv[i]} items {cnt[i]} {ms[i]:.2f} ms "
          f"{fl[i]/max(ms[i],1e-9)/1e9:.2f} TF/s")
# per-launch dump for offline analysis: kind, level, items, ms, flops, bytes
import os
os.makedirs("gpurun_out", exist_ok=True)
np.savetxt(f"gpurun_out/launch_dump_{N}_{form}.csv",
           np.column_stack([kinds, lv, cnt, ms, fl, by]), delimiter=",",
           header="kind,level,items,ms,flops,bytes", fmt=["%d", "%d", "%d", "%.6f", "%.6e", "%.6e"])
