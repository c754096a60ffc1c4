"""Aggregate per-tile timings of the DMMA update launches (debug, non-graph).

  python tools/tile_stats.py N"""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, ".")
os.environ["PS_KEEP_TILES"] = "1"
from paper_1405_2636_b200 import sparse
from paper_1405_2636_b200.analysis import analyze, AnalyzeOptions
from paper_1405_2636_b200.pipeline import get_engine, default_pivot_threshold
from paper_1405_2636_b200._native import ptr
N = int(sys.argv[1]) if len(sys.argv) > 1 else 60
an = analyze(sparse.gen_laplacian(3, (N, N, N)), AnalyzeOptions())
eng = get_engine(an)
thr = default_pivot_threshold(an.A_perm)
n = ctypes.c_int64()
eng.lib.ps_plan_tile_count(eng.handle, ctypes.byref(n))
nt = n.value
T = np.zeros((nt, 24), dtype=np.int32)
eng._check(eng.lib.ps_plan_tiles(eng.handle, ptr(T)))
dtr = torch.zeros(3 * nt, dtype=torch.int64, device="cuda")
eng._check(eng.lib.ps_set_tile_trace(eng.handle, ctypes.c_void_p(dtr.data_ptr())))
store = eng.new_store()
for _ in range(2):
    eng.assemble(store, an.A_perm)
    tb = eng.factor_timed(store, "llt", thr, per_launch=True)
eng.check("llt")
tr = dtr.cpu().numpy().reshape(nt, 3).astype(np.int64)
kinds, lv, cnt = eng.launch_table()
first = 0
rows = []
for i, k in enumerate(kinds):
    if k in (2, 3, 4):
        a, b = first, first + cnt[i]
        first = b
        t = tr[a:b]
        ok = t[:, 0] > 0
        if not ok.any():
            continue
        body = (t[ok, 1] - t[ok, 0]) / 1e3
        tail = (t[ok, 2] - t[ok, 1]) / 1e3
        span = (t[ok, 2].max() - t[ok, 0].min()) / 1e3
        kn = T[a:b, 7][ok]
        rows.append((k, lv[i], b - a, span, tb["per_launch_ms"][i] * 1e3, body.mean(), tail.mean(), kn.mean(),
                     (2.0 * T[a:b, 4] * T[a:b, 5] * T[a:b, 7]).sum()))
rows = np.array(rows)
for k, name in ((2, "trail (intra)"), (3, "update (inter)"), (4, "narrow")):
    r = rows[rows[:, 0] == k]
    print(f"{name}: launches {len(r)} sum launch {r[:,4].sum()/1e3:.2f} ms, sum span {r[:,3].sum()/1e3:.2f} ms, "
          f"tile body mean {np.average(r[:,5], weights=r[:,2]):.2f} us, epilogue mean {np.average(r[:,6], weights=r[:,2]):.2f} us, "
          f"mean K {np.average(r[:,7], weights=r[:,2]):.0f}, flops {r[:,8].sum():.3g} -> {r[:,8].sum()/r[:,4].sum()/1e6:.2f} TF/s")
    # by tile count bucket
    for lo, hi in ((0, 64), (64, 256), (256, 1024), (1024, 10**9)):
        m = (r[:, 2] >= lo) & (r[:, 2] < hi)
        if m.any():
            print(f"   tiles [{lo},{hi}): launches {m.sum()} sum launch {r[m,4].sum()/1e3:.2f} ms, mean launch {r[m,4].mean():.1f} us, "
                  f"mean body {np.average(r[m,5], weights=r[m,2]):.2f} us, mean K {np.average(r[m,7], weights=r[m,2]):.0f}")
