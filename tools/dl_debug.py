import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_1405_2636_b200 import sparse
from paper_1405_2636_b200.analysis import analyze
from paper_1405_2636_b200.pipeline import factorize
an = analyze(sparse.gen_laplacian(3, (40, 40, 40)))
r = factorize(an)
h = r.store.slab.copy(); d = r.device_store.tensor.cpu().numpy()
s = an.symbol
so = s.storage_offsets; off = np.asarray(so() if callable(so) else so); w = np.asarray(s.widths); nr = np.asarray(s.nrows_arr); print("off", off.shape, off[:3])
bad = np.flatnonzero(h != d)
print("differing entries", len(bad), "of", len(h))
if len(bad):
    ps = np.unique(np.searchsorted(off, bad, side="right") - 1)
    print("panels", len(ps), "first", [(int(p), int(w[p]), int(nr[p])) for p in ps[:10]])
    p = ps[0]; loc = bad[(bad >= off[p]) & (bad < off[p+1])] - off[p]
    cols = np.unique(loc // nr[p]); print("cols of first bad panel", cols[:20], "...", len(cols))
    for p in ps[:6]:
        loc = bad[(bad >= off[p]) & (bad < off[p+1])] - off[p]
        print("panel", int(p), "w", int(w[p]), "nr", int(nr[p]), "bad", len(loc), "cols", np.unique(loc // nr[p])[:8], "rows", np.unique(loc % nr[p])[:8])
