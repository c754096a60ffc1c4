"""Narrow-tile timeline per launch (debug): preamble (start -> before the
color wait), wait, RMW + signal; per-CTA serial tiles."""
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
n = ctypes.c_int64(); eng.lib.ps_plan_tile_count(eng.handle, ctypes.byref(n)); nt = n.value
T = np.zeros((nt, 17), dtype=np.int32); eng._check(eng.lib.ps_plan_tiles(eng.handle, ptr(T)))
dtr = torch.zeros(3 * nt, dtype=torch.int64, device="cuda")
eng._check(eng.lib.ps_set_tile_trace(eng.handle, ctypes.c_void_p(dtr.data_ptr())))
st = eng.new_store(); eng.assemble(st, an.A_perm)
tb = eng.factor_timed(st, "llt", default_pivot_threshold(an.A_perm), per_launch=True); eng.check("llt")
tr = dtr.cpu().numpy().reshape(nt, 3).astype(np.int64)
kinds, lv, cnt = eng.launch_table()
first = 0; rng = {}
for i, k in enumerate(kinds):
    if k in (2, 3, 4):
        rng[i] = (first, first + cnt[i]); first += cnt[i]
for i in [i for i in rng if kinds[i] == 4][:12]:
    a, b = rng[i]
    t = tr[a:b]
    ok = t[:, 2] > 0
    t = t[ok]
    t0 = t[:, 0].min()
    pre = (t[:, 1] - t[:, 0]) / 1e3; post = (t[:, 2] - t[:, 1]) / 1e3
    span = (t[:, 2].max() - t0) / 1e3
    print(f"launch {i} level {lv[i]}: {b-a} tiles span {span:.1f} us (event {tb['per_launch_ms'][i]*1e3:.1f}); "
          f"preamble mean {pre.mean():.2f} us, wait+rmw+signal mean {post.mean():.2f} max {post.max():.1f}; "
          f"tiles/CTA-slot ~{(b-a)/1036:.1f}")
