"""Where the time goes in the public-API path factorize(an) + .store (dev tool)."""
import sys, time
import torch
sys.path.insert(0, ".")
from paper_1405_2636_b200 import sparse
from paper_1405_2636_b200.analysis import analyze, AnalyzeOptions
from paper_1405_2636_b200.pipeline import get_engine, default_pivot_threshold, factorize, DeviceStore
N = int(sys.argv[1]) if len(sys.argv) > 1 else 60
A = sparse.gen_laplacian(3, (N, N, N))
an = analyze(A, AnalyzeOptions())
for _ in range(3):
    r = factorize(an); _ = r.store.slab[0]
def T(f, *a):
    torch.cuda.synchronize(); t = time.perf_counter(); out = f(*a); torch.cuda.synchronize(); return out, (time.perf_counter() - t) * 1e3
eng = get_engine(an)
_, t1 = T(default_pivot_threshold, an.A_perm)
_, t2 = T(eng.new_store)
dv, t3 = T(eng.upload_values, an.A_perm)
st = eng.new_store()
_, t4 = T(eng.assemble, st, an.A_perm, dv)
_, t5 = T(lambda: (eng.factor(st, "llt", 1e-13), eng.check("llt")))
r, t6 = T(factorize, an)
_, t7 = T(lambda: r.store)
r2, t8 = T(factorize, an)
_, t9 = T(lambda: r2.store.slab[0])
print(f"thr {t1:.1f} new_store {t2:.1f} upload {t3:.1f} assemble {t4:.1f} factor+check {t5:.1f} | factorize {t6:.1f} to_host {t7:.1f} | again factorize {t8:.1f} to_host {t9:.1f} ms; pool {[len(v) for v in DeviceStore._pool.values()]}")
