"""Calibrate the stratified CPU sample against one full oracle run (60^3 LLt).

    python tools/cpu_calibrate.py > profiles/r02_cpu_calibration.json
"""
import json
import os
import sys
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from oracle import panel_oracle as O  # noqa: E402
from oracle.cpu_sample import run_sample  # noqa: E402
from paper_1405_2636_b200 import sparse  # noqa: E402
from paper_1405_2636_b200.analysis import analyze  # noqa: E402
from paper_1405_2636_b200.symbolic import allocate_panels  # noqa: E402

size = int(sys.argv[1]) if len(sys.argv) > 1 else 60
an = analyze(sparse.gen_laplacian(3, (size, size, size)))
store = allocate_panels(an.symbol, an.A_perm)
t = time.perf_counter()
O.factorize(an.symbol, store, "llt", O.pivot_threshold(an.A_perm))
full = time.perf_counter() - t
est = run_sample(os.path.join(ROOT, "bench_data", f"cpu_sample_{size}_llt.npz"), 1)
ref = np.load(os.path.join(ROOT, "tests", "golden", f"big_lap3d_{size}_llt.npz"))
print(json.dumps({
    "config": f"LLT 3D 7-point Laplacian {size}^3, 1 BLAS thread, this build container",
    "flops": an.flops,
    "oracle_full_run_s": full, "oracle_full_gflops": an.flops / full / 1e9,
    "reference_full_run_s": float(ref["factor_s"]),
    "reference_full_gflops": an.flops / float(ref["factor_s"]) / 1e9,
    "stratified_estimate_s": est["est_seconds_1core"],
    "stratified_gflops": est["gflops_per_core"],
    "sample_seconds": est["sampled_seconds"],
    "estimate_over_full_oracle": full / est["est_seconds_1core"],
    "estimate_over_reference": float(ref["factor_s"]) / est["est_seconds_1core"],
}, indent=1))
