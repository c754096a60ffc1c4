"""Drop-in numeric pipeline: factorize() on the B200 engine, solve, report.

Mirrors the reference's `pipeline.factorize` / `FactorResult` /
`run_report` / `check_solve` (pipeline.py:73-156).  Every scheduler name
the reference accepts ("dynamic", "static", "sequential") and "gpu" run the
same CUDA engine - the CPU task runtime is what this package replaces;
`threads`, `kernel` and `deterministic` are accepted for signature
compatibility (the engine is always deterministic).  `wall_seconds` times
the numeric phase only, on the device (CUDA events), as the reference times
pipeline.py:97-116.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import sparse
from .analysis import Analysis, AnalyzeOptions, analyze  # noqa: F401  (re-export)
from .errors import DeviceError
from .solve import supernodal_solve
from .symbolic import PanelStore

SCHEDULERS = ("gpu", "dynamic", "static", "sequential")


_DIAG_POS = []  # (colptr, rowidx, positions) of recently used patterns (most recent last)


def diagonal_positions(A):
    """Positions of A's diagonal entries in A.values (cached per pattern: the
    colptr / rowidx arrays are taken as immutable; the values may change)."""
    for cp, ri, pos in _DIAG_POS:
        if cp is A.colptr and ri is A.rowidx:
            return pos
    pos = np.flatnonzero(A.rowidx == A.entry_cols())
    _DIAG_POS.append((A.colptr, A.rowidx, pos))
    del _DIAG_POS[:-4]
    return pos


def default_pivot_threshold(A):
    """1e-13 * max |diag(A)| (reference kernels.py:32-40), from the current
    values on every call."""
    if A.n == 0 or A.nnz == 0:
        return 0.0
    pos = diagonal_positions(A)
    if len(pos) == 0:
        return 0.0
    return 1e-13 * float(np.abs(A.values[pos]).max())


def _resolve_device(device):
    """torch.device('cuda', index) for None / 'cuda' / 'cuda:k' / torch.device."""
    import torch
    dev = torch.device(device if device is not None else "cuda")
    if dev.type != "cuda":
        raise DeviceError(f"the B200 engine runs on CUDA devices, not {dev}")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    return dev


def get_engine(analysis, device=None):
    """The (cached) device plan of an analysis, one per CUDA device."""
    from .engine import Engine
    device = _resolve_device(device)
    cache = analysis.__dict__.setdefault("_engines", {})
    key = device.index
    eng = cache.get(key)
    if eng is None:
        eng = Engine(analysis.symbol, device)
        cache[key] = eng
    return eng


class DeviceStore:
    """Factored slab resident on the GPU; host PanelStore on demand.

    The pinned host slab comes from a per-size pool and goes back to it when
    this object is garbage-collected, so repeated factorize() + read cycles
    do not pay a pinned allocation of the whole factor each time."""

    _pool = {}

    def __init__(self, symbol, tensor):
        self.symbol = symbol
        self.tensor = tensor
        self._host = None
        self._uhost = None
        self._pinned = None

    @staticmethod
    def pinned_slab(n, dtype=None):
        """A pinned host slab of n values from the per-(size, dtype) pool."""
        import torch
        dtype = dtype or torch.float64
        free = DeviceStore._pool.setdefault((n, dtype), [])
        return free.pop() if free else torch.empty(n, dtype=dtype, pin_memory=True)

    def _download(self):
        import torch
        if self._pinned is None:  # not downloaded alongside the factorization
            host = DeviceStore.pinned_slab(self.tensor.numel(), self.tensor.dtype)
            host.copy_(self.tensor, non_blocking=True)
            self._pinned = host
        torch.cuda.current_stream(self.tensor.device).synchronize()
        return self._pinned.numpy()

    def to_host(self):
        """The L factor (the reference's PanelStore layout; LU: L with U's
        diagonal, the first of the two slabs)."""
        if self._host is None:
            h = self._download()
            e = int(self.symbol.storage_offsets()[-1])
            self._host = PanelStore(self.symbol, slab=h[:e] if h.size != e else h)
            if h.size == 2 * e:
                self._uhost = PanelStore(self.symbol, slab=h[e:])
        return self._host

    def to_host_u(self):
        """LU: U transposed in the same layout (u[r, j] = U[fc + j, row r])."""
        self.to_host()
        return self._uhost

    def __del__(self):
        # recycle only when nothing else still sees the host slab (the
        # PanelStore or any numpy view of it)
        try:
            import sys
            h = self._host
            key = None if self._pinned is None else (self._pinned.numel(), self._pinned.dtype)
            if self._pinned is not None and h is None:  # downloaded, never viewed
                DeviceStore._pool.setdefault(key, []).append(self._pinned)
            elif (self._pinned is not None and h is not None and self._uhost is None
                    and sys.getrefcount(h) == 3 and sys.getrefcount(h.data) == 2
                    and sys.getrefcount(h.slab) == 3):
                DeviceStore._pool.setdefault(key, []).append(self._pinned)
        except Exception:
            pass


@dataclass
class FactorResult:
    analysis: Analysis
    device_store: DeviceStore
    form: str
    _events: list = None
    wall_seconds: float = 0.0
    schedule: object = None
    _trace: object = None

    @property
    def events(self):
        """The reference's TraceEvent list (runtime.py:28-36): one event per
        task of the DAG, from a timed replay of the same factorization
        (collect_trace=True; taken on first access so that the timed
        factorization itself runs as one CUDA graph).  [] otherwise."""
        if self._events is None:
            self._events = self._trace() if self._trace is not None else []
            self._trace = None
        return self._events

    @property
    def store(self):
        """Host PanelStore (reference layout; downloaded once)."""
        return self.device_store.to_host()

    @property
    def ustore(self):
        """LU only: the U factor, transposed into the PanelStore layout."""
        return self.device_store.to_host_u() if self.form == "lu" else None

    def solve(self, b, refine=0):
        """x with A x = b from the factor (reference FactorResult.solve,
        pipeline.py:82-84 -> supernodal_solve, kernels.py:332-382), on the GPU
        when the factor is device-resident (ps_solve).  refine > 0: that many
        steps of iterative refinement with the same factor."""
        b = np.asarray(b)
        if self.device_store is not None and self.device_store.tensor.is_complex():
            b = b.astype(np.complex128)
        elif np.iscomplexobj(b):  # real factor: real and imaginary parts separately
            return self.solve(b.real, refine) + 1j * self.solve(b.imag, refine)
        else:
            b = b.astype(np.float64)
        if self.device_store is None:
            x = supernodal_solve(self.analysis.symbol, self.store, b, self.form,
                                 self.analysis.perm.perm)
            for _ in range(refine):
                r = b - _spmv_original(self.analysis, x)
                x = x + supernodal_solve(self.analysis.symbol, self.store, r, self.form,
                                         self.analysis.perm.perm)
            return x
        x = self._gpu_solve(b)
        for _ in range(refine):
            x = x + self._gpu_solve(b - _spmv_original(self.analysis, x))
        return x

    def _gpu_solve(self, b):
        import torch
        t = self.device_store.tensor
        an = self.analysis
        eng = get_engine(an, t.device)
        perm = an.__dict__.get("_perm_dev")
        if perm is None or perm.device != t.device:
            perm = torch.from_numpy(np.ascontiguousarray(an.perm.perm, dtype=np.int64)).to(t.device)
            an.__dict__["_perm_dev"] = perm
        bd = torch.from_numpy(np.ascontiguousarray(b)).to(t.device)
        x = torch.empty_like(bd)
        x[perm] = bd
        stream = torch.cuda.current_stream(t.device)
        eng.solve(t, x, self.form, stream=stream)
        return x[perm].cpu().numpy()


def factorize(analysis, scheduler="gpu", threads=1, kernel="buffered", deterministic=False,
              collect_trace=True, device=None, download=True):
    """Numeric factorization of an analyzed matrix on the B200 engine.

    download=True (default) also moves the factor into a pinned host slab,
    overlapped with the factorization (each slab chunk as soon as it is
    final), so `FactorResult.store` (the reference's host PanelStore) costs
    no separate copy; download=False keeps the factor on the device only
    (GPU solve), and `.store` then copies on first access."""
    if scheduler not in SCHEDULERS:
        raise ValueError(f"unknown scheduler '{scheduler}'")
    if threads == 0:
        raise ValueError("threads must be >= 1")
    import torch
    form = analysis.options.form
    eng = get_engine(analysis, device)
    store = eng.new_store(form, analysis.is_complex)
    stream = torch.cuda.current_stream(eng.device)
    dvals = eng.upload_values(analysis.A_perm, stream=stream)
    eng.assemble(store, analysis.A_perm, dvals, stream=stream, form=form)
    # the pivot threshold of pipeline.py:88-91, every call from the current
    # values: NaN asks the engine for the reference default 1e-13 max|diag(A)|
    # from the assembled slab on the device (no host round trip before the
    # factorization is enqueued)
    thr = float("nan")
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    ds = DeviceStore(analysis.symbol, store)
    t0.record(stream)
    if download:
        ds._pinned = DeviceStore.pinned_slab(store.numel(), store.dtype)
        eng.factor_download(store, form, thr, ds._pinned, stream=stream)
    else:
        eng.factor(store, form, thr, stream=stream)
    t1.record(stream)
    eng.check(form, stream=stream)
    wall = t0.elapsed_time(t1) / 1e3
    trace = ((lambda: _trace_events(analysis, eng, form, default_pivot_threshold(analysis.A_perm)))
             if collect_trace else None)
    return FactorResult(analysis, ds, form, None, wall, None, trace)


def _trace_events(analysis, eng, form, thr):
    """Per-task GPU timeline of a replay of the factorization (scratch slab)."""
    from .trace import events_from_timeline
    import torch
    stream = torch.cuda.current_stream(eng.device)
    store = eng.new_store(form, analysis.is_complex)
    eng.assemble(store, analysis.A_perm, eng.upload_values(analysis.A_perm, stream=stream),
                 stream=stream, form=form)
    tl = eng.timeline(store, form, thr, stream=stream)
    del store
    return events_from_timeline(analysis.symbol, eng, tl["start_ms"], tl["per_launch_ms"])


@dataclass
class RunReport:
    matrix: str
    n: int
    nnz_a: int
    nnz_l: int
    flops: int
    scheduler: str
    threads: int
    wall_seconds: float
    gflops: float
    residual: float | None
    status: str

    CSV_HEADER = ("matrix,n,nnz_a,nnz_l,flops,scheduler,threads,"
                  "wall_s,gflops,residual,status")

    def csv_row(self):
        res = "" if self.residual is None else f"{self.residual:.3e}"
        return (f"{self.matrix},{self.n},{self.nnz_a},{self.nnz_l},{self.flops},"
                f"{self.scheduler},{self.threads},{self.wall_seconds:.6f},"
                f"{self.gflops:.3f},{res},{self.status}")


def run_report(name, A, result, scheduler, threads, residual=None, status="ok"):
    an = result.analysis
    wall = result.wall_seconds
    gflops = an.flops / wall / 1e9 if wall > 0 else 0.0
    return RunReport(name, an.symbol.n, an.nnz_a, an.symbol.nnz_l, an.flops, scheduler,
                     threads, wall, gflops, residual, status)


def _spmv_original(analysis, x):
    """A x in the original ordering from the permuted lower storage
    (A_perm[perm[i], perm[j]] = A[i, j])."""
    perm = analysis.perm.perm
    xp = np.empty_like(x)
    xp[perm] = x
    return sparse.spmv(analysis.A_perm, xp)[perm]


def check_solve(A, result):
    """Scaled residual of b = A @ ones (reference pipeline.py:152-156)."""
    b = sparse.spmv(A, np.ones(A.n))
    x = result.solve(b)
    return sparse.residual_norm(A, x, b), x
