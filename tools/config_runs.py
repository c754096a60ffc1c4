"""Every BASELINE.json config that fits one GPU: factorization time and rate
(reference flop model, same symbol), raw backward error ||Ax-b||/||b|| with
b = A 1 and after one step of iterative refinement with the same factors
(SURVEY 0.6).  Writes gpurun_out/configs.json.

  python tools/config_runs.py [names...]   (default: all)"""
import json, os, sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1405_2636_b200 import sparse
from paper_1405_2636_b200.analysis import analyze, AnalyzeOptions
from paper_1405_2636_b200.pipeline import get_engine, default_pivot_threshold, DeviceStore
from paper_1405_2636_b200.solve import supernodal_solve

CONFIGS = {
    "C1_2d64_llt": (2, 64, "llt", 0.0),
    "C2_3d60_llt": (3, 60, "llt", 0.0),
    "C3_3d80_ldlt_shift": (3, 80, "ldlt", 0.5),
    "C5_3d120_llt": (3, 120, "llt", 0.0),
}
names = sys.argv[1:] or list(CONFIGS)
out = {}
for name in names:
    dim, N, form, shift = CONFIGS[name]
    A = sparse.gen_laplacian(dim, (N,) * dim)
    if shift:
        A = sparse.shift_diagonal(A, shift)
    t = time.time(); an = analyze(A, AnalyzeOptions(form=form)); t_an = time.time() - t
    t = time.time(); eng = get_engine(an); t_plan = time.time() - t
    thr = default_pivot_threshold(an.A_perm)
    store = eng.new_store()
    best = 1e30
    for _ in range(4):
        eng.assemble(store, an.A_perm)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); eng.factor(store, form, thr); e1.record(); eng.check(form)
        best = min(best, e0.elapsed_time(e1))
    from paper_1405_2636_b200.pipeline import FactorResult
    res = FactorResult(an, DeviceStore(an.symbol, store), form, [], best / 1e3, None)
    b = sparse.spmv(A, np.ones(A.n))
    x = res.solve(b)  # GPU solve (ps_solve), warm
    torch.cuda.synchronize()
    t = time.time()
    x = res.solve(b)
    t_solve = time.time() - t
    raw = sparse.backward_error(A, x, b)
    x1 = res.solve(b, refine=1)
    ref1 = sparse.backward_error(A, x1, b)
    out[name] = {"n": A.n, "form": form, "flops": int(an.flops), "factor_ms": best,
                 "gflops": an.flops / best / 1e6, "fp64_peak_frac": an.flops / best / 1e6 / 37.1e3,
                 "backward_error_raw": raw, "backward_error_refined_1step": ref1,
                 "analyze_s": t_an, "plan_s": t_plan, "gpu_solve_s": t_solve,
                 "panels": int(an.symbol.npanels), "nnz_l": int(an.symbol.nnz_l)}
    print(name, json.dumps(out[name]), flush=True)
    del store, res
    eng.close()
    an.__dict__.pop("_engines", None)
    torch.cuda.empty_cache()
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/configs.json", "w"), indent=1)
