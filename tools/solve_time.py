"""GPU solve time (dev tool): python tools/solve_time.py N"""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1405_2636_b200 import sparse
from paper_1405_2636_b200.analysis import analyze, AnalyzeOptions
from paper_1405_2636_b200.pipeline import factorize
N = int(sys.argv[1]) if len(sys.argv) > 1 else 60
A = sparse.gen_laplacian(3, (N, N, N))
an = analyze(A, AnalyzeOptions())
res = factorize(an)
b = sparse.spmv(A, np.ones(A.n))
x = res.solve(b)
torch.cuda.synchronize()
t = time.time(); x = res.solve(b); torch.cuda.synchronize(); dt = time.time() - t
print(f"N={N} solve {dt*1e3:.1f} ms berr {sparse.backward_error(A, x, b):.2e}")
from paper_1405_2636_b200.pipeline import get_engine
eng = get_engine(an)
xd = torch.from_numpy(b).cuda()
for _ in range(2):
    eng.solve(res.device_store.tensor, xd, "llt")
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); eng.solve(res.device_store.tensor, xd, "llt"); e1.record(); torch.cuda.synchronize()
print(f"ps_solve device time {e0.elapsed_time(e1):.2f} ms")
t = time.time(); _ = res._gpu_solve(b); torch.cuda.synchronize(); print(f"_gpu_solve {1e3*(time.time()-t):.1f} ms")
