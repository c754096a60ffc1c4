"""Sampled reference factors at the BASELINE configurations (C2, C3, C5).

Run in the build container only (imports the reference from
/root/reference, which does not exist on the GPU box); each case is one
process so the three can run side by side:

    PYTHONPATH=/root/reference/pkg/src OPENBLAS_NUM_THREADS=1 \
        python tests/golden/make_golden_big.py lap3d_60_llt

Output (committed): tests/golden/big_<case>.npz with
  sample        slab[::stride] of the reference's factor (panel order, each
                panel F-order -- the PanelStore layout, symbolic.py:318-335)
  stride        the sampling stride (a prime, ~1e5 entries per file)
  chunk_norm    Frobenius norm of each of 8192 equal contiguous slab chunks
                (every entry of the factor enters one of them)
  max_abs       max |L| over the whole slab
  flops, digest symbol flop count / digest (the same symbol as ours)
  berr          ||A x - b|| / ||b|| for b = A 1 (pipeline.py:152-156)
  factor_s      reference factor wall time (sequential, 1 BLAS thread)
  spread        (LDLt only) max|L_seq - L_dyn| / max|L_seq|, the reference's
                own schedule-to-schedule spread (dynamic, 8 threads)
"""

import os
import sys
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")
import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(__file__))
from panelsolve import pipeline, sparse  # noqa: E402  (the reference)
from make_golden import digest_of, shifted, slab_of  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
NCHUNK = 8192

CASES = {
    "lap3d_40_llt": (40, 0.0, "llt"),
    "lap3d_60_llt": (60, 0.0, "llt"),
    "lap3d_80_ldlt_shift": (80, 0.5, "ldlt"),
    "lap3d_120_llt": (120, 0.0, "llt"),
}


def _prime_at_least(x):
    x = max(int(x), 3) | 1
    while any(x % d == 0 for d in range(3, int(x ** 0.5) + 1, 2)):
        x += 2
    return x


def chunk_norms(slab, nchunk=NCHUNK):
    edges = np.linspace(0, slab.size, nchunk + 1).astype(np.int64)
    return np.array([np.linalg.norm(slab[a:b]) for a, b in zip(edges[:-1], edges[1:])])


def stream(store, npanels, stride):
    """sample / chunk norms / max without concatenating the slab (120^3: 13 GB)."""
    size = sum(store.data[p].size for p in range(npanels))
    edges = np.linspace(0, size, NCHUNK + 1).astype(np.int64)
    sq = np.zeros(NCHUNK)
    samples, pos, mx = [], 0, 0.0
    for p in range(npanels):
        v = store.data[p].ravel(order="F")
        first = (-pos) % stride
        samples.append(v[first::stride])
        mx = max(mx, float(np.abs(v).max()) if v.size else 0.0)
        c0 = np.searchsorted(edges, pos, "right") - 1
        c1 = np.searchsorted(edges, pos + v.size, "right") - 1
        for c in range(c0, min(c1, NCHUNK - 1) + 1):
            a, b = max(edges[c], pos) - pos, min(edges[c + 1], pos + v.size) - pos
            if b > a:
                sq[c] += float(np.dot(v[a:b], v[a:b]))
        pos += v.size
    return np.concatenate(samples), np.sqrt(sq), mx, size


def main(case):
    N, shift, form = CASES[case]
    A = sparse.gen_laplacian(3, (N, N, N))
    if shift:
        A = shifted(A, shift)
    t = time.time()
    an = pipeline.analyze(A, pipeline.AnalyzeOptions(form=form))
    ta = time.time() - t
    print(case, "analyze", ta, flush=True)
    t = time.time()
    res = pipeline.factorize(an, "sequential")
    tf = time.time() - t
    print(case, "factor", tf, flush=True)
    _, x = pipeline.check_solve(A, res)
    b = sparse.spmv(A, np.ones(A.n))
    berr = float(np.linalg.norm(sparse.spmv(A, x) - b) / np.linalg.norm(b))
    npan = an.symbol.npanels
    size = sum(res.store.data[p].size for p in range(npan))
    stride = _prime_at_least(size / 100000)
    sample, cn, mx, size = stream(res.store, npan, stride)
    out = dict(sample=sample, stride=stride, chunk_norm=cn, max_abs=mx, flops=int(an.flops),
               digest=digest_of(an), berr=berr, factor_s=tf, analyze_s=ta,
               size=size, form=form, shift=shift, N=N)
    if form == "ldlt":
        slab = slab_of(an, res.store)
        del res
        t = time.time()
        r2 = pipeline.factorize(an, "dynamic", threads=8, collect_trace=False)
        print(case, "dynamic", time.time() - t, flush=True)
        s2 = slab_of(an, r2.store)
        out["spread"] = float(np.abs(slab - s2).max() / np.abs(slab).max())
        cn2 = chunk_norms(s2)
        out["spread_chunk"] = float(np.max(np.abs(cn2 - cn) / np.maximum(cn, 1e-300)))
    np.savez_compressed(os.path.join(HERE, f"big_{case}.npz"), **out)
    print(case, "done", {k: v for k, v in out.items() if np.ndim(v) == 0}, flush=True)


if __name__ == "__main__":
    main(sys.argv[1])
