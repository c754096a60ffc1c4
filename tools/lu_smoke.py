import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_1405_2636_b200 import sparse
from paper_1405_2636_b200.analysis import analyze, AnalyzeOptions
from paper_1405_2636_b200.pipeline import factorize, get_engine
from oracle import panel_oracle_ext as X
def rel(a, b): return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))
for N in (6, 12):
    A = sparse.gen_convdiff27(N)
    Ac = sparse.gen_convdiff27(N, complex_shift=1.0)
    for name, B, form in [("lu", A, "lu"), ("lu_c", Ac, "lu"), ("llt_c", sparse.symmetrize_pattern(Ac), "llt"),
                          ("ldlt_c", sparse.symmetrize_pattern(Ac), "ldlt"),
                          ("ldlt_shift_c", sparse.shift_diagonal(sparse.symmetrize_pattern(Ac), 30.0), "ldlt")]:
        an = analyze(B, AnalyzeOptions(form=form))
        res = factorize(an)
        st, ut = X.factor_analysis(an)
        e1 = rel(res.store.slab, st.slab)
        e2 = rel(res.ustore.slab, ut.slab) if form == "lu" else 0.0
        b = sparse.spmv(B, np.ones(B.n) + (0.5j if np.iscomplexobj(B.values) else 0))
        x = res.solve(b)
        print(N, name, an.symbol.max_width(), "L", e1, "U", e2, "berr", sparse.backward_error(B, x, b), flush=True)
# generic real llt/ldlt vs tuned
A = sparse.gen_laplacian(3, (14, 14, 14))
for form in ("llt", "ldlt"):
    B = A if form == "llt" else sparse.shift_diagonal(A, 0.5)
    an = analyze(B, AnalyzeOptions(form=form))
    r1 = factorize(an).store.slab.copy()
    eng = get_engine(an); eng.generic = True
    r2 = factorize(an)
    x = r2.solve(sparse.spmv(B, np.ones(B.n)))
    eng.generic = False
    print("generic", form, rel(r2.store.slab, r1), sparse.backward_error(B, x, sparse.spmv(B, np.ones(B.n))))
