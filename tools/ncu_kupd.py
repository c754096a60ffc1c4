"""Non-graph factorization for an ncu capture of the heaviest k_update launch.

  python tools/ncu_kupd.py N info [L]    -> prints level, tiles, ordinal (k_update launches in
                                            table order) and the ncu --launch-skip to use
                                            (heaviest launch, or heaviest of level L)
  python tools/ncu_kupd.py N run         -> one warm-up + one timed non-graph factorization"""
import json, sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1405_2636_b200 import sparse
from paper_1405_2636_b200.analysis import analyze, AnalyzeOptions
from paper_1405_2636_b200.pipeline import get_engine, default_pivot_threshold
N = int(sys.argv[1]) if len(sys.argv) > 1 else 60
mode = sys.argv[2] if len(sys.argv) > 2 else "info"
an = analyze(sparse.gen_laplacian(3, (N, N, N)), AnalyzeOptions())
eng = get_engine(an)
thr = default_pivot_threshold(an.A_perm)
kinds, lv, cnt = eng.launch_table()
lflops, lbytes = eng.launch_work()
# launches that run the k_update kernel itself: K_UPDATE launches of at least
# sms * 3 tiles (smaller ones run k_update8, trailing tiles k_trail8) unless
# the 8-warp kernels are switched off
import os
sms = torch.cuda.get_device_properties(0).multi_processor_count
# (and of mean tile K >= 64: ps_b200.cu PS_U8_KEFF)
is_ku = (kinds == 3) & (cnt >= sms * 3) & (lflops >= 64 * 2.0 * 64 * 64 * cnt)
if os.environ.get("PS_TRAIL8") == "0":
    is_ku |= kinds == 2
ku = np.flatnonzero(is_ku)
best = int(np.argmax(lflops[ku]))
if len(sys.argv) > 3:  # a given level: its heaviest k_update launch
    lev = int(sys.argv[3])
    cand = [j for j in range(len(ku)) if lv[ku[j]] == lev]
    best = max(cand, key=lambda j: lflops[ku[j]])
idx = int(ku[best])
if mode == "info":
    print(json.dumps({"level": int(lv[idx]), "tiles": int(cnt[idx]), "ordinal": best,
                      "launch_skip": len(ku) + best, "flops": float(lflops[idx]),
                      "alg_bytes": float(lbytes[idx])}))
else:
    store = eng.new_store()
    for _ in range(2):
        eng.assemble(store, an.A_perm)
        eng.factor_timed(store, "llt", thr)
    torch.cuda.synchronize()
