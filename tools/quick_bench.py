"""Quick device timing of the factorization (development tool, not bench.py)."""
import sys, time
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
t = time.time(); an = analyze(A, AnalyzeOptions(form=form)); ta = time.time() - t
t = time.time(); eng = get_engine(an); tp = time.time() - t
print(f"N={N} form={form} analyze {ta:.2f}s plan {tp:.2f}s info {eng.info}", flush=True)
thr = default_pivot_threshold(an.A_perm)
store = eng.new_store()
s = torch.cuda.current_stream()
for it in range(6):
    eng.assemble(store, an.A_perm)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); eng.factor(store, form, thr); e1.record()
    eng.check(form)
    ms = e0.elapsed_time(e1)
    print(f"iter {it}: {ms:.3f} ms  {an.flops / ms / 1e6:.1f} GFlop/s", flush=True)
eng.assemble(store, an.A_perm)
tb = eng.factor_timed(store, form, thr)
print("timed breakdown", tb, flush=True)
eng.assemble(store, an.A_perm)
eng.factor(store, form, thr); eng.check(form)
from paper_1405_2636_b200.pipeline import DeviceStore
from paper_1405_2636_b200.solve import supernodal_solve
hs = DeviceStore(an.symbol, store).to_host()
b = sparse.spmv(A, np.ones(A.n))
x = supernodal_solve(an.symbol, hs, b, form, an.perm.perm)
print("backward error", sparse.backward_error(A, x, b), "residual", sparse.residual_norm(A, x, b))
