"""CPU baseline on a stratified sample - TEST / BENCH INFRASTRUCTURE ONLY.

Times the oracle's restatement of the reference kernels (panel_oracle:
factor_panel = kernels.py:208-247, update_couple = kernels.py:128-136 and
249-281) on the units of a sample drawn by tools/make_cpu_sample.py (one
unit = one panel's factor task plus every update task it sources), then
extrapolates per width class:

    T_est = sum_s F_s * (sampled time_s / sampled flops_s)
    GFlop/s = total flops / T_est

It reads only the sample file (numpy arrays); no analysis, no native
library of this repository.  Values are synthetic but well conditioned
(diagonally dominant diagonal blocks), so no pivot fails and no denormals
slow the BLAS.  workers > 1 runs the units concurrently in that many
processes (one BLAS thread each; per-unit times include the contention) and
reports workers x the extrapolated per-core rate: an ideally parallel CPU
runtime, an upper bound for the reference, whose multi-threaded schedulers
run slower than its sequential one.
"""

from __future__ import annotations

import os
import time

import numpy as np

from . import panel_oracle as O


class _MiniSymbol:
    def __init__(self, z):
        self.starts = z["fc"]
        self.widths = z["w"]
        self.blkptr = z["blkptr"]
        self.blk_fr = z["blk_fr"]
        self.blk_lr = z["blk_lr"]
        self.blk_facing = z["blk_facing"]
        self.blk_loc = z["blk_loc"]


class _Panels:
    """Panel arrays created on first use (a worker allocates only its own
    units' sources and destinations; 120^3 destinations reach 1.6 GB)."""

    def __init__(self, z, rng):
        self.z, self.rng, self.cache = z, rng, {}

    def __getitem__(self, i):
        a = self.cache.get(i)
        if a is None:
            z = self.z
            wi = int(z["w"][i])
            m = int(z["rowptr"][i + 1] - z["rowptr"][i])
            a = np.asfortranarray(self.rng.uniform(-1e-3, 1e-3, (wi + m, wi)))
            a[np.arange(wi), np.arange(wi)] = 1.0 + wi * 1e-3
            self.cache[i] = a
        return a


class _Rowmaps:
    def __init__(self, z):
        self.z = z

    def __getitem__(self, i):
        z = self.z
        fc, w, rp = int(z["fc"][i]), int(z["w"][i]), z["rowptr"]
        return np.concatenate([np.arange(fc, fc + w), z["rows"][rp[i]:rp[i + 1]]])


class _MiniStore:
    def __init__(self, z, rng):
        self.data = _Panels(z, rng)
        self.rowmaps = _Rowmaps(z)


def _run_units(path, units, form):
    """Per-unit seconds of the given source units (one process, 1 BLAS thread)."""
    try:
        from threadpoolctl import threadpool_limits
        lim = threadpool_limits(limits=1)
    except Exception:  # pragma: no cover
        lim = None
    z = dict(np.load(path))
    sym = _MiniSymbol(z)
    store = _MiniStore(z, np.random.default_rng(1))
    out = []
    with np.errstate(all="ignore"):
        for i in units:  # allocate outside the timed region
            store.data[i]
            for b in range(int(sym.blkptr[i]), int(sym.blkptr[i + 1])):
                store.data[int(sym.blk_facing[b])]
            t = time.perf_counter()
            O.factor_panel(store.data[i], int(sym.starts[i]), form, -np.inf)
            b0, b1 = int(sym.blkptr[i]), int(sym.blkptr[i + 1])
            groups = {}
            for b in range(b0, b1):
                groups.setdefault(int(sym.blk_facing[b]), []).append(b)
            for q in sorted(groups):
                O.update_couple(sym, store, i, q, groups[q], form)
            out.append(time.perf_counter() - t)
    del lim
    return out


def _worker(args):
    return _run_units(*args)


def run_sample(path, workers=1):
    """Estimated reference CPU rate (GFlop/s) of the whole factorization."""
    z = np.load(path)
    nsrc = int(z["nsrc"])
    form = str(z["form"])
    cls = z["src_class"]
    fl = z["src_flops"]
    t0 = time.perf_counter()
    if workers <= 1:
        secs = np.array(_run_units(path, list(range(nsrc)), form))
    else:
        import multiprocessing as mp
        order = np.argsort(-fl)  # heaviest first, dealt round-robin
        parts = [order[k::workers].tolist() for k in range(workers)]
        ctx = mp.get_context("spawn")
        with ctx.Pool(workers) as pool:
            res = pool.map(_worker, [(path, p, form) for p in parts])
        secs = np.zeros(nsrc)
        for p, r in zip(parts, res):
            secs[p] = r
    wall = time.perf_counter() - t0
    F = z["class_flops"]
    t_est = 0.0
    per_class = []
    for c in range(len(F)):
        m = cls == c
        if F[c] == 0:
            continue
        rate = fl[m].sum() / secs[m].sum()  # flops per second of this class
        t_est += F[c] / rate
        per_class.append({"widths": [int(z["strata"][c]), int(z["strata"][c + 1]) - 1],
                          "units": int(m.sum()), "of": int(z["class_units"][c]),
                          "gflops": rate / 1e9, "share_of_flops": float(F[c] / z["total_flops"])})
    gflops_1core = float(z["total_flops"]) / t_est / 1e9
    # workers > 1: the units ran concurrently (shared memory bandwidth and
    # caches), an ideally parallel runtime divides the single-core time
    return {"gflops": gflops_1core * max(1, workers),
            "gflops_per_core": gflops_1core, "est_seconds_1core": t_est,
            "sampled_seconds": float(secs.sum()), "wall_seconds": wall, "workers": workers,
            "units": nsrc, "sampled_flops": float(fl.sum()),
            "total_flops": float(z["total_flops"]), "classes": per_class}
