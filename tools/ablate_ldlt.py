"""80^3 shifted LDLt factor timing without the status check (dev tool)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_1405_2636_b200 import sparse
from paper_1405_2636_b200.analysis import analyze, AnalyzeOptions
from paper_1405_2636_b200.pipeline import get_engine, default_pivot_threshold
N = int(sys.argv[1]) if len(sys.argv) > 1 else 80
A = sparse.shift_diagonal(sparse.gen_laplacian(3, (N, N, N)), 0.5)
an = analyze(A, AnalyzeOptions(form="ldlt"))
eng = get_engine(an)
thr = default_pivot_threshold(an.A_perm)
store = eng.new_store()
ts = []
for it in range(6):
    eng.assemble(store, an.A_perm)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); eng.factor(store, "ldlt", thr); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ts = sorted(ts[2:])
print(f"N={N} ldlt factor median {ts[len(ts)//2]:.3f} ms min {ts[0]:.3f}")
