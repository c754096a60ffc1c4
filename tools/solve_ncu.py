"""One GPU solve between cudaProfilerStart/Stop (dev tool), for
ncu --profile-from-start off ... python tools/solve_ncu.py N"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1405_2636_b200 import sparse
from paper_1405_2636_b200.analysis import analyze, AnalyzeOptions
from paper_1405_2636_b200.pipeline import factorize, get_engine
N = int(sys.argv[1]) if len(sys.argv) > 1 else 60
A = sparse.gen_laplacian(3, (N, N, N))
an = analyze(A, AnalyzeOptions())
res = factorize(an)
eng = get_engine(an)
xd = torch.from_numpy(sparse.spmv(A, np.ones(A.n))).cuda()
eng.solve(res.device_store.tensor, xd.clone(), "llt")
torch.cuda.synchronize()
torch.cuda.profiler.start()
eng.solve(res.device_store.tensor, xd.clone(), "llt")
torch.cuda.synchronize()
torch.cuda.profiler.stop()
