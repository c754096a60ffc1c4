"""Generate the golden fixtures from the REFERENCE implementation.

Run in the build container only (it imports the reference from
/root/reference, which does not exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src OPENBLAS_NUM_THREADS=1 \
        python tests/golden/make_golden.py [--big]

Outputs (committed):
  tests/golden/factors_small.npz  reference factor slabs (panel order, each
                                  panel F-order) for small configurations
  tests/golden/golden.json        symbol digests, flop counts, residuals,
                                  sampled factor entries for larger ones
"""

import json
import os
import sys
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(__file__))
from panelsolve import kernels, pipeline, sparse  # noqa: E402  (the reference)
from digest import symbol_digest  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def slab_of(an, store):
    return np.concatenate([store.data[p].ravel(order="F") for p in range(an.symbol.npanels)])


def digest_of(an):
    sym = an.symbol
    starts = [p.fc for p in sym.panels] + [sym.n]
    rows = np.concatenate([p.rows for p in sym.panels]) if sym.npanels else []
    blocks = np.array([(b.fr, b.lr, b.facing, b.loc) for p in sym.panels for b in p.blocks],
                      dtype=np.int64).reshape(-1, 4)
    return symbol_digest(starts, rows, blocks, an.perm.perm)


def shifted(A, s):
    vals = A.values.copy()
    cols = np.repeat(np.arange(A.n), np.diff(A.colptr))
    vals[A.rowidx == cols] -= s
    return sparse.SparseMatrix(A.n, A.colptr, A.rowidx, vals, "symmetric-lower")


def rand_spd(rng, n, density):
    mask = np.tril(rng.random((n, n)) < density, -1)
    vals = rng.uniform(-1.0, 1.0, (n, n)) * mask
    Ad = vals + vals.T
    Ad += np.diag(np.abs(Ad).sum(axis=1) + rng.uniform(0.5, 1.5, n))
    r, c = np.nonzero(np.tril(Ad))
    return sparse.from_coo(n, r, c, Ad[r, c], "symmetric-lower")


def small_cases():
    rng = np.random.default_rng(20240211)
    yield "lap2d_16_llt", sparse.gen_laplacian(2, (16, 16)), "llt"
    yield "lap2d_64_llt", sparse.gen_laplacian(2, (64, 64)), "llt"
    yield "lap3d_8_llt", sparse.gen_laplacian(3, (8, 8, 8)), "llt"
    yield "lap3d_8_ldlt_shift", shifted(sparse.gen_laplacian(3, (8, 8, 8)), 0.5), "ldlt"
    yield "lap2d_16_ldlt_shift", shifted(sparse.gen_laplacian(2, (16, 16)), 0.5), "ldlt"
    yield "rand_spd_120", rand_spd(rng, 120, 0.15), "llt"
    yield "rand_spd_60_ldlt", rand_spd(rng, 60, 0.3), "ldlt"


def main(big=False):
    out = {}
    slabs = {}
    meta = {}
    for name, A, form in small_cases():
        an = pipeline.analyze(A, pipeline.AnalyzeOptions(form=form))
        res = pipeline.factorize(an, "sequential")
        slabs[name] = slab_of(an, res.store)
        r, _ = pipeline.check_solve(A, res)
        meta[name] = {"form": form, "flops": int(an.flops), "digest": digest_of(an),
                      "residual": float(r), "n": int(an.symbol.n),
                      "npanels": int(an.symbol.npanels)}
        print(name, meta[name]["flops"], len(slabs[name]))
    np.savez_compressed(os.path.join(HERE, "factors_small.npz"), **slabs)
    out["small"] = meta
    # larger: digests, flops, residuals, sampled entries, LDLt self-spread
    large = {}
    sizes = [24] + ([40, 60] if big else [])
    for N in sizes:
        A = sparse.gen_laplacian(3, (N, N, N))
        t = time.time()
        an = pipeline.analyze(A)
        ta = time.time() - t
        t = time.time()
        res = pipeline.factorize(an, "sequential")
        tf = time.time() - t
        r, x = pipeline.check_solve(A, res)
        b = sparse.spmv(A, np.ones(A.n))
        berr = float(np.linalg.norm(sparse.spmv(A, x) - b) / np.linalg.norm(b))
        slab = slab_of(an, res.store)
        step = 101
        ent = {"digest": digest_of(an), "flops": int(an.flops), "nnz_l": int(an.symbol.nnz_l),
               "npanels": int(an.symbol.npanels), "nblocks": int(an.symbol.block_count()),
               "residual": float(r), "backward_error": berr, "analyze_s": ta, "factor_s": tf,
               "max_abs_L": float(np.abs(slab).max()), "sample_step": step,
               "sample": slab[::step].tolist() if N <= 24 else None}
        large[f"lap3d_{N}_llt"] = ent
        print(N, "llt", ent["flops"], tf)
    # shifted LDLt at 24^3: the reference's own sequential-vs-dynamic spread
    A = shifted(sparse.gen_laplacian(3, (24, 24, 24)), 0.5)
    an = pipeline.analyze(A, pipeline.AnalyzeOptions(form="ldlt"))
    r1 = pipeline.factorize(an, "sequential")
    r2 = pipeline.factorize(an, "dynamic", threads=8)
    s1, s2 = slab_of(an, r1.store), slab_of(an, r2.store)
    rr, x = pipeline.check_solve(A, r1)
    b = sparse.spmv(A, np.ones(A.n))
    large["lap3d_24_ldlt_shift"] = {
        "digest": digest_of(an), "flops": int(an.flops), "residual": float(rr),
        "backward_error": float(np.linalg.norm(sparse.spmv(A, x) - b) / np.linalg.norm(b)),
        "self_spread": float(np.abs(s1 - s2).max() / np.abs(s1).max()),
        "max_abs_L": float(np.abs(s1).max()), "sample_step": 101,
        "sample": s1[::101].tolist()}
    out["large"] = large
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main(big="--big" in sys.argv)
