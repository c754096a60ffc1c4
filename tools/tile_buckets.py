"""All DMMA update tiles of one factorization: body time by tile size (debug)."""
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
T = np.zeros((nt, 24), dtype=np.int32); eng._check(eng.lib.ps_plan_tiles(eng.handle, ptr(T)))
dtr = torch.zeros(3 * nt, dtype=torch.int64, device="cuda")
eng._check(eng.lib.ps_set_tile_trace(eng.handle, ctypes.c_void_p(dtr.data_ptr())))
st = eng.new_store(); eng.assemble(st, an.A_perm)
eng.factor_timed(st, "llt", default_pivot_threshold(an.A_perm)); eng.check("llt")
tr = dtr.cpu().numpy().reshape(nt, 3).astype(np.int64)
ok = tr[:, 2] > 0
body = (tr[:, 2] - tr[:, 0]) / 1e3
fl = 2.0 * T[:, 4] * T[:, 5] * T[:, 7]
intra = T[:, 8] < 0
for name, sel0 in (("inter", ~intra), ("intra", intra)):
    sel = sel0 & ok
    print(f"{name}: {sel.sum()} tiles, CTA-time {body[sel].sum()/1e3:.1f} ms, flops {fl[sel].sum():.3e}")
    edges = [0, 1e4, 1e5, 3e5, 1e6, 3e6, 1e12]
    for a, b in zip(edges[:-1], edges[1:]):
        m = sel & (fl >= a) & (fl < b)
        if m.any():
            print(f"   flops [{a:.0e},{b:.0e}): n {m.sum():7d} mean {body[m].mean():6.1f} us  CTA-time {body[m].sum()/1e3:8.1f} ms "
                  f"({body[m].sum()/body[sel].sum():5.1%})  {fl[m].sum()/body[m].sum()/1e3:6.1f} GF/s/CTA  K mean {T[m,7].mean():.0f}")
