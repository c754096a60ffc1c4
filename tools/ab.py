"""A/B timing of engine variants on ONE box, interleaved (development tool).

    python tools/ab.py N form lib_a.so lib_b.so [...]   (form: llt | ldlt | lu)

Each variant library (tools/build_var.sh NAME "-D...") gets its own plan of
the same analysis; rounds alternate between the variants, each round timing
3 graph-replayed factorizations (assembly + factor, CUDA events).  Prints
the median ms per variant and checks the variants' factors agree.
"""
import ctypes
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_1405_2636_b200 import _abi, _native, engine as _eng, sparse  # noqa: E402
from paper_1405_2636_b200.analysis import AnalyzeOptions, analyze  # noqa: E402
from paper_1405_2636_b200.pipeline import default_pivot_threshold  # noqa: E402

N, form, libs = int(sys.argv[1]), sys.argv[2], sys.argv[3:]
if form in ("lu", "luc"):  # luc: complex LU
    A = sparse.gen_convdiff27(N, complex_shift=1.0 if form == "luc" else None)
    form = "lu"
else:
    A = sparse.gen_laplacian(3, (N, N, N))
    if form == "ldlt":
        A = sparse.shift_diagonal(A, 0.5)
an = analyze(A, AnalyzeOptions(form=form))
thr = default_pivot_threshold(an.A_perm)
engines = []
import os
for spec in libs:  # lib.so[:VAR=value,VAR2=value] - env knobs read at plan creation
    path, _, envs = spec.partition(":")
    for kv in filter(None, envs.split(",")):
        k, v = kv.split("=")
        os.environ[k] = v
    lib = _abi.bind(ctypes.CDLL(path))
    _eng.engine_lib = lambda lib=lib: lib
    e = _eng.Engine(an.symbol)
    st = e.new_store(form, an.is_complex)
    dv = e.upload_values(an.A_perm)
    for kv in filter(None, envs.split(",")):
        os.environ.pop(kv.split("=")[0], None)
    engines.append((spec, e, st, dv))
times = {p: [] for p in libs}
for rnd in range(5):
    for path, e, st, dv in engines:
        for _ in range(3 if rnd else 1):
            e.assemble(st, an.A_perm, dv, form=form)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            e.factor(st, form, thr)
            e1.record()
            try:
                e.check(form)
            except Exception as ex:  # timing-only variants (wrong results) still time
                if rnd == 0:
                    print(f"{path}: check failed: {ex}", flush=True)
            if rnd:
                times[path].append(e0.elapsed_time(e1))
ref = engines[0][2]
for path, e, st, dv in engines:
    ms = statistics.median(times[path])
    d = float((st - ref).abs().max() / ref.abs().max())
    print(f"{path}: median {ms:.3f} ms ({an.flops / ms / 1e6:.0f} GFlop/s), "
          f"min {min(times[path]):.3f}, max|d| vs first {d:.2e}", flush=True)
