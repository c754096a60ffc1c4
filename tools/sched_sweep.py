"""Factorization time for schedule variants (env set by the caller), dev tool."""
import os, sys
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
best = 1e9
for _ in range(5):
    eng.assemble(store, an.A_perm)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); eng.factor(store, form, thr); e1.record(); eng.check(form)
    best = min(best, e0.elapsed_time(e1))
tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("PS_"))
print(f"N={N} {form} [{tag}] {best:.3f} ms {an.flops/best/1e9:.2f} TF/s", flush=True)
