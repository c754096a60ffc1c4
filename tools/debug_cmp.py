"""Per-panel comparison of the GPU factor with the oracle (debug tool)."""
import os, sys, time
import numpy as np
sys.path.insert(0, ".")
import torch
from paper_1405_2636_b200 import sparse
from paper_1405_2636_b200.analysis import analyze
from paper_1405_2636_b200.pipeline import factorize
from oracle import panel_oracle as O
N = int(sys.argv[1])
A = sparse.gen_laplacian(3, (N, N, N))
an = analyze(A)
res = factorize(an)
g = res.store
t = time.time(); r = O.factor_analysis(an); print("oracle s", time.time() - t, flush=True)
sym = an.symbol
par = sym.panel_parent()
lev = np.zeros(sym.npanels, dtype=int)
for p in range(sym.npanels):
    if par[p] >= 0: lev[par[p]] = max(lev[par[p]], lev[p] + 1)
off = sym.storage_offsets()
bad = []
for p in range(sym.npanels):
    a, b = g.slab[off[p]:off[p+1]], r.slab[off[p]:off[p+1]]
    e = np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)
    if e > 1e-10: bad.append((p, e))
print("bad panels", len(bad))
for p, e in bad[:15]:
    print(p, f"err {e:.3e} w {sym.widths[p]} nrows {sym.nrows_arr[p]} level {lev[p]} nblk {sym.blkptr[p+1]-sym.blkptr[p]}")
