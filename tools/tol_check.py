import sys, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from _cases import small_cases
from paper_1405_2636_b200.analysis import AnalyzeOptions, analyze
from paper_1405_2636_b200.pipeline import factorize
import test_gpu_parity as T
for name, A, form in small_cases():
    an = analyze(A, AnalyzeOptions(form=form))
    res = factorize(an)
    print(name, form, f"{T.rel(res.store.slab, T.SLABS[name]):.2e}")
