"""One factorization (CUDA-graph replay) for ncu launch lists / captures.

  python tools/ncu_one.py [N] [form] [reps]
Runs analysis + plan, one warm-up factorization, then `reps` factorizations."""
import sys
import torch
sys.path.insert(0, ".")
from paper_1405_2636_b200 import sparse
from paper_1405_2636_b200.analysis import analyze, AnalyzeOptions
from paper_1405_2636_b200.pipeline import get_engine, default_pivot_threshold

N = int(sys.argv[1]) if len(sys.argv) > 1 else 60
form = sys.argv[2] if len(sys.argv) > 2 else "llt"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
A = sparse.gen_laplacian(3, (N, N, N))
if form == "ldlt":
    A = sparse.shift_diagonal(A, 0.5)
an = analyze(A, AnalyzeOptions(form=form))
eng = get_engine(an)
thr = default_pivot_threshold(an.A_perm)
store = eng.new_store()
for _ in range(reps):
    eng.assemble(store, an.A_perm)
    eng.factor(store, form, thr)
    eng.check(form)
torch.cuda.synchronize()
print("launches per factorization", eng.launches_per_factorization)
