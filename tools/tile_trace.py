"""Per-tile timeline of the level schedule's DMMA update launches (debug).

  PS_KEEP_TILES=1 python tools/tile_trace.py N [launch ...]"""
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
eng.assemble(store, an.A_perm)
tb = eng.factor_timed(store, "llt", thr, per_launch=True)
eng.check("llt")
tr = dtr.cpu().numpy().reshape(nt, 3)
kinds, lv, cnt = eng.launch_table()
# tile ranges per launch (K_UPDATE=3 and K_TRAIL=2 share the tile array, in launch order)
first = 0
ranges = {}
for i, k in enumerate(kinds):
    if k in (2, 3, 4):
        ranges[i] = (first, first + cnt[i])
        first += cnt[i]
want = []
for a in sys.argv[2:]:  # launch index, or L<level>: that level's longest DMMA update launch
    if a.startswith("L"):
        sel = (kinds == 3) & (lv == int(a[1:]))
        want.append(int(np.argmax(np.where(sel, tb["per_launch_ms"], -1))))
    else:
        want.append(int(a))
want = want or [int(np.argmax(np.where(kinds == 3, tb["per_launch_ms"], 0)))]
for L in want:
    a, b = ranges[L]
    t = tr[a:b].astype(np.int64)
    t0 = t[:, 0].min()
    st, ml, en = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3, (t[:, 2] - t0) / 1e3
    tl = T[a:b]
    work = 2.0 * tl[:, 4] * tl[:, 5] * tl[:, 7]
    print(f"launch {L} (kind {kinds[L]}, level {lv[L]}): {b-a} tiles, span {en.max():.1f} us, launch event {tb['per_launch_ms'][L]*1e3:.1f} us")
    print(f"  tile body (start->mainloop done) mean {np.mean(ml-st):.1f} max {np.max(ml-st):.1f} us; wait+epilogue mean {np.mean(en-ml):.1f} max {np.max(en-ml):.1f}")
    print(f"  useful rate {work.sum() / (en.max() * 1e-6) / 1e12:.2f} TFLOP/s; K histogram {dict(zip(*np.unique(tl[:, 7], return_counts=True)))}" if len(tl) < 0 else
          f"  useful rate {work.sum() / (en.max() * 1e-6) / 1e12:.2f} TFLOP/s; kn median {np.median(tl[:, 7]):.0f}, full tiles {np.mean((tl[:, 4] == 64) & (tl[:, 5] == 64)):.2f}")
    print(f"  start times: 50% {np.median(st):.1f} 90% {np.quantile(st,0.9):.1f} max {st.max():.1f} us")
    late = np.argsort(-en)[:8]
    for k in late:
        print(f"   tail tile {a+k}: src {tl[k,0]} dst {tl[k,1]} ni {tl[k,4]} nj {tl[k,5]} kn {tl[k,7]} wait {tl[k,9]} "
              f"start {st[k]:.1f} ml {ml[k]:.1f} end {en[k]:.1f} flops {work[k]:.3g}")
    heavy = np.argsort(-work)[:5]
    for k in heavy:
        print(f"   heavy tile {a+k}: kn {tl[k,7]} start {st[k]:.1f} ml {ml[k]:.1f} end {en[k]:.1f} us")
