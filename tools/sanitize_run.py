"""One small factorization + GPU solve through the public API, for
compute-sanitizer (tests/test_gpu_sanitizer.py):

    compute-sanitizer --tool racecheck python tools/sanitize_run.py 12 llt
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1405_2636_b200 import sparse  # noqa: E402
from paper_1405_2636_b200.analysis import AnalyzeOptions, analyze  # noqa: E402
from paper_1405_2636_b200.pipeline import factorize  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 12
form = sys.argv[2] if len(sys.argv) > 2 else "llt"
if form == "lu":
    A = sparse.gen_convdiff27(N)
else:
    A = sparse.gen_laplacian(3, (N, N, N))
    if form == "ldlt":
        A = sparse.shift_diagonal(A, 0.5)
an = analyze(A, AnalyzeOptions(form=form))
res = factorize(an)
b = sparse.spmv(A, np.ones(A.n))
berr = sparse.backward_error(A, res.solve(b, refine=1), b)
print(f"sanitize_run N={N} {form}: backward error {berr:.2e}")
sys.exit(0 if berr <= 1e-12 else 1)
