"""GPU engine: a Python handle over the C-ABI plan (include/ps_b200.h).

Device memory and streams come from PyTorch (plumbing); all numeric work is
in the sm_100a kernels of libps_b200.so.  There is no CPU fallback - if the
library or a CUDA device is missing, construction raises.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _abi
from ._native import engine_lib, ptr
from .errors import (DeviceError, NotPositiveDefiniteError, SingularPivotError,
                     StructuralError)
from .symbolic import assembly_positions, assembly_positions_lu


def _torch():
    import torch
    return torch


def _stream_handle(stream):
    torch = _torch()
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


class HostRegistry:
    """Per-process page-locking of host arrays (ps_host_register), keyed by
    address and size.  A registration lives as long as its array: it is
    released (after the last copy out of it has completed) when the array is
    garbage-collected.  Arrays that cannot be registered (read-only, shared
    pages, already pinned elsewhere is fine) are remembered so that the
    registration is not retried on every call."""

    _live = {}     # (ptr, nbytes) -> [weakref finalizer, last copy event, owned]
    _failed = set()

    @classmethod
    def pin(cls, lib, v):
        key = (v.ctypes.data, v.nbytes)
        if key in cls._live:
            return True
        if key in cls._failed:
            return False
        reg = ctypes.c_int(0)
        if lib.ps_host_register(ctypes.c_void_p(key[0]), key[1], ctypes.byref(reg)) != 0 \
                or reg.value == 0:
            cls._failed.add(key)
            return False
        import weakref
        ent = [None, None, reg.value == 1]
        ent[0] = weakref.finalize(v, cls._release, lib, key)
        cls._live[key] = ent
        return True

    @classmethod
    def after_copy(cls, v, stream):
        ent = cls._live.get((v.ctypes.data, v.nbytes))
        if ent is not None:
            ev = _torch().cuda.Event()
            ev.record(stream)
            ent[1] = ev

    @classmethod
    def _release(cls, lib, key):
        ent = cls._live.pop(key, None)
        if ent is None:
            return
        if ent[1] is not None:
            ent[1].synchronize()  # the DMA out of the range has finished
        if ent[2]:
            lib.ps_host_unregister(ctypes.c_void_p(key[0]))


class Engine:
    """Factorization plan for one symbol on one CUDA device.

    A plan serves one call at a time; calls on different streams are
    serialized by the library (each waits for the previous call's work)."""

    def __init__(self, symbol, device=None, partition=None, top_owner=None):
        torch = _torch()
        if not torch.cuda.is_available():
            raise DeviceError("the B200 engine needs a CUDA device (no CPU fallback)")
        self.lib = engine_lib()
        dev = torch.device(device if device is not None else "cuda")
        if dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        self.symbol = symbol
        s = symbol
        self._keep = [np.ascontiguousarray(a, dtype=np.int64) for a in
                      (s.starts, s.rowptr, s.rowdata, s.blkptr, s.blk_fr, s.blk_lr,
                       s.blk_facing, s.blk_loc)]
        k = self._keep
        desc = _abi.SymbolDesc(s.n, s.npanels, *[ptr(a) for a in k])
        h = ctypes.c_void_p()
        with torch.cuda.device(dev):
            if partition is None:
                rc = self.lib.ps_plan_create(ctypes.byref(desc), dev.index, ctypes.byref(h))
            elif top_owner is None:
                grp, ngroups, mine = partition
                self._group = np.ascontiguousarray(grp, dtype=np.int32)
                rc = self.lib.ps_plan_create_partitioned(ctypes.byref(desc), dev.index,
                                                         ptr(self._group), int(ngroups),
                                                         int(mine), ctypes.byref(h))
            else:
                grp, ngroups, mine = partition
                self._group = np.ascontiguousarray(grp, dtype=np.int32)
                self._owner = np.ascontiguousarray(top_owner, dtype=np.int32)
                rc = self.lib.ps_plan_create_distributed(ctypes.byref(desc), dev.index,
                                                         ptr(self._group), int(ngroups),
                                                         int(mine), ptr(self._owner),
                                                         ctypes.byref(h))
        self._check(rc)
        self.handle = h
        info = _abi.PlanInfo()
        self._check(self.lib.ps_plan_get_info(h, ctypes.byref(info)))
        self.info = {f: getattr(info, f) for f, _ in _abi.PlanInfo._fields_}
        self.offsets = np.empty(s.npanels + 1, dtype=np.int64)
        self._check(self.lib.ps_plan_offsets(h, ptr(self.offsets)))
        self._assembly = None

    # ------------------------------------------------------------------
    def _err(self):
        m = self.lib.ps_last_error()
        return m.decode() if m else ""

    def _check(self, rc, form=None, col=None, piv=None):
        if rc == _abi.PS_OK:
            return
        if rc == _abi.PS_NUMERIC:
            if form in ("ldlt", "lu"):
                raise SingularPivotError(int(col), float(piv))
            raise NotPositiveDefiniteError(int(col), float(piv))
        if rc == _abi.PS_STRUCTURAL:
            raise StructuralError(self._err())
        raise DeviceError(f"engine error {rc}: {self._err()}")

    def close(self):
        if getattr(self, "handle", None):
            self.lib.ps_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------
    @property
    def store_elems(self):
        return int(self.info["store_elems"])

    generic = False  # tests: real LLt / LDLt on the scalar-generic kernels

    def code(self, form, store=None, complex_=None):
        """ABI form code (ps_b200.h): the form, | complex (from the store's
        dtype unless given), | generic (self.generic)."""
        if complex_ is None:
            complex_ = store is not None and store.is_complex()
        return _abi.form_code(form, complex_, self.generic)

    def new_store(self, form="llt", complex_=False):
        """Device slab(s) of the factor: store_elems values, twice for LU (the
        L slab, then the U slab), complex128 for complex values."""
        torch = _torch()
        n = self.store_elems * (2 if form == "lu" else 1)
        return torch.empty(n, dtype=torch.complex128 if complex_ else torch.float64,
                           device=self.device)

    def assembly(self, A_perm):
        """Device copy of the slab position of A_perm's entries (analysis-time;
        cached) and the host selection mask of the lower entries.  General
        (LU) matrices: every entry, upper ones into the U slab."""
        if self._assembly is None or self._assembly[0] is not A_perm:
            torch = _torch()
            if A_perm.stype == "general":
                full = assembly_positions_lu(self.symbol, A_perm)
                sel = np.ones(len(full), dtype=bool)
                dfull = torch.from_numpy(full).to(self.device)
                self._assembly = (A_perm, dfull, sel, dfull)
            else:
                pos, sel = assembly_positions(self.symbol, A_perm)
                dpos = torch.from_numpy(pos).to(self.device)
                full = np.full(len(sel), -1, dtype=np.int64)  # every entry of A: -1 = upper
                full[sel] = pos
                self._assembly = (A_perm, dpos, sel, torch.from_numpy(full).to(self.device))
        return self._assembly[1], self._assembly[2]

    def _host_values(self, A_perm):
        """A_perm.values as a page-locked CPU tensor: the array itself,
        registered once per process (HostRegistry), else a copy into a
        pinned staging buffer."""
        torch = _torch()
        v = A_perm.values
        if v.dtype in (np.float64, np.complex128) and v.flags.c_contiguous and v.size and \
                HostRegistry.pin(self.lib, v):
            return torch.from_numpy(v)
        dt = torch.complex128 if np.iscomplexobj(v) else torch.float64
        pin = getattr(self, "_pin_stage", None)
        if pin is None or pin.numel() != v.size or pin.dtype != dt:
            pin = torch.empty(v.size, dtype=dt, pin_memory=True)
            self._pin_stage = pin
        np.copyto(pin.numpy(), v)
        return pin

    def upload_values(self, A_perm, stream=None):
        """H2D of all of A's values from page-locked host memory (no host-side
        gather: the assembly skips the upper entries on the device).  The
        host array must stay unchanged until `stream` has passed the copy;
        its registration is released only after the copy has completed."""
        torch = _torch()
        self.assembly(A_perm)
        src = self._host_values(A_perm)
        dvals = torch.empty(src.numel(), dtype=src.dtype, device=self.device)
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        with torch.cuda.stream(s):
            dvals.copy_(src, non_blocking=True)
        HostRegistry.after_copy(A_perm.values, s)
        return dvals

    def assemble(self, store, A_perm, dvals=None, stream=None, form=None):
        """Zero the slab(s) and scatter A's values (device assembly): the lower
        ones (symmetric forms) or all of them, upper ones into the U slab (LU)."""
        torch = _torch()
        dpos, sel = self.assembly(A_perm)
        if form is None:
            form = "lu" if A_perm.stype == "general" else "llt"
        if dvals is None:
            vals = np.ascontiguousarray(A_perm.values[sel])
            dvals = torch.from_numpy(vals).to(self.device, non_blocking=False)
        elif dvals.numel() == len(sel) and dvals.numel() != dpos.numel():
            dpos = self._assembly[3]  # all entries (upload_values): upper ones skipped
        rc = self.lib.ps_assemble_form(self.handle, ctypes.c_void_p(store.data_ptr()),
                                       ctypes.c_void_p(dpos.data_ptr()),
                                       ctypes.c_void_p(dvals.data_ptr()), int(dvals.numel()),
                                       self.code(form, store), _stream_handle(stream))
        self._check(rc)

    def factor(self, store, form, thr, stream=None, phase=-1):
        """Enqueue the factorization (CUDA graph replay); asynchronous.
        phase 0 / 1: the rank-local part / the top of a partitioned plan."""
        rc = self.lib.ps_factor_phase(self.handle, ctypes.c_void_p(store.data_ptr()),
                                      self.code(form, store), float(thr), _stream_handle(stream),
                                      int(phase))
        self._check(rc)

    def factor_download(self, store, form, thr, host, stream=None):
        """Enqueue the factorization plus the download of the factor slab
        into the pinned host tensor `host`, overlapped: each slab chunk is
        copied as soon as its last writing launch has run (ps_factor_download).
        Asynchronous; a synchronize of `stream` covers the copies."""
        rc = self.lib.ps_factor_download(self.handle, ctypes.c_void_p(store.data_ptr()),
                                         self.code(form, store), float(thr),
                                         _stream_handle(stream), ctypes.c_void_p(host.data_ptr()))
        self._check(rc)

    def assemble_positions(self, store, dpos, dvals, stream=None):
        """Zero the slab and scatter explicit (position, value) pairs."""
        rc = self.lib.ps_assemble(self.handle, ctypes.c_void_p(store.data_ptr()),
                                  ctypes.c_void_p(dpos.data_ptr()),
                                  ctypes.c_void_p(dvals.data_ptr()), int(dvals.numel()),
                                  _stream_handle(stream))
        self._check(rc)

    KIND_NAMES = ("factor_w1", "factor_small", "update_intra", "update_dmma",
                  "update_narrow", "factor_diag_inv", "trsm_dmma", "(unused)",
                  "(unused)", "join", "fork", "xwait")

    def launch_table(self, branches=False):
        """(kind, level, count[, branch]) of every launch of a factorization."""
        n = int(self.info["nlaunches"])
        k = np.zeros(n, dtype=np.int32)
        lv = np.zeros(n, dtype=np.int32)
        c = np.zeros(n, dtype=np.int32)
        br = np.zeros(n, dtype=np.int32)
        self._check(self.lib.ps_plan_launches(self.handle, ptr(k), ptr(lv), ptr(c), ptr(br)))
        return (k, lv, c, br) if branches else (k, lv, c)

    def segments(self):
        """Distributed-top plans: (bounds[nseg + 1], levels[nseg]) of the phase-1 segments."""
        n = ctypes.c_int32()
        self._check(self.lib.ps_plan_segments(self.handle, None, None, ctypes.byref(n)))
        b = np.zeros(n.value + 1, dtype=np.int32)
        lv = np.zeros(max(1, n.value), dtype=np.int32)
        self._check(self.lib.ps_plan_segments(self.handle, ptr(b), ptr(lv), ctypes.byref(n)))
        return b, lv[:n.value]

    def factor_range(self, store, form, thr, i0, i1, stream=None):
        rc = self.lib.ps_factor_range(self.handle, ctypes.c_void_p(store.data_ptr()),
                                      self.code(form, store), float(thr), _stream_handle(stream),
                                      int(i0), int(i1))
        self._check(rc)

    def status_all(self, stream=None):
        self._check(self.lib.ps_factor_status_all(self.handle, _stream_handle(stream)))

    def launch_work(self):
        """(flops, algorithmic bytes) of every level-schedule launch."""
        n = len(self.launch_table()[0])
        f = np.zeros(max(1, n))
        b = np.zeros(max(1, n))
        self._check(self.lib.ps_plan_launch_work(self.handle, ptr(f), ptr(b)))
        return f[:n], b[:n]

    def factor_timed(self, store, form, thr, stream=None, per_launch=False):
        """Non-graph run with events around every launch: ms per kernel kind
        (and, with per_launch, the per-launch milliseconds)."""
        ms = np.zeros(3)
        nl = np.zeros(1, dtype=np.int32)
        pl = np.zeros(max(1, int(self.info["nlaunches"])), dtype=np.float32)
        rc = self.lib.ps_factor_timed(self.handle, ctypes.c_void_p(store.data_ptr()),
                                      self.code(form, store), float(thr), _stream_handle(stream),
                                      ptr(ms), ptr(nl), ptr(pl))
        self._check(rc)
        out = {"factor_ms": float(ms[0]), "trailing_ms": float(ms[1]),
               "update_ms": float(ms[2]), "launches": int(nl[0])}
        if per_launch:
            out["per_launch_ms"] = pl[:int(nl[0])].astype(np.float64)
        return out

    def timeline(self, store, form, thr, stream=None):
        """Serialized run with events around every launch: per-launch start
        and duration (ms), relative to the first launch (ps_factor_timeline)."""
        n = max(1, int(self.info["nlaunches"]))
        pl = np.zeros(n, dtype=np.float32)
        st = np.zeros(n, dtype=np.float32)
        nl = np.zeros(1, dtype=np.int32)
        rc = self.lib.ps_factor_timeline(self.handle, ctypes.c_void_p(store.data_ptr()),
                                         self.code(form, store), float(thr),
                                         _stream_handle(stream), None, ptr(nl), ptr(pl), ptr(st))
        self._check(rc)
        k = int(nl[0])
        return {"start_ms": st[:k].astype(np.float64), "per_launch_ms": pl[:k].astype(np.float64)}

    def check(self, form, stream=None):
        """Synchronize and raise the reference's exception on pivot failure."""
        col = ctypes.c_int64(0)
        piv = ctypes.c_double(0.0)
        rc = self.lib.ps_factor_status(self.handle, _stream_handle(stream), ctypes.byref(col),
                                       ctypes.byref(piv))
        self._check(rc, form, col.value, piv.value)

    def solve(self, store, x, form, stream=None):
        """In-place supernodal solve of the device vector x (PERMUTED order)
        with the factor in `store` (ps_solve; reference kernels.py:332-382)."""
        if x.is_complex() != store.is_complex():
            raise ValueError("solve: the right-hand side and the factor must both be real or complex")
        rc = self.lib.ps_solve(self.handle, ctypes.c_void_p(store.data_ptr()),
                               ctypes.c_void_p(x.data_ptr()), self.code(form, store),
                               _stream_handle(stream))
        self._check(rc)

    # per-task operators (reference plugin protocol, kernels.py:311-315)
    def run_factor_task(self, store, p, form, thr, stream=None):
        rc = self.lib.ps_run_factor_task(self.handle, ctypes.c_void_p(store.data_ptr()), int(p),
                                         self.code(form, store), float(thr),
                                         _stream_handle(stream))
        self._check(rc)
        self.check(form, stream)

    def run_update_task(self, store, p, q, form, stream=None):
        rc = self.lib.ps_run_update_task(self.handle, ctypes.c_void_p(store.data_ptr()), int(p),
                                         int(q), self.code(form, store), _stream_handle(stream))
        self._check(rc)

    @property
    def launches_per_factorization(self):
        # kernel launches of ps_factor: the per-level launches (branch-join
        # markers excluded) + the status reduction
        n = int(self.info["nlaunches"])
        if self.info["nlaunches"] > 1:
            n -= int(np.isin(self.launch_table()[0], (9, 10, 11)).sum())
        return n + (1 if self.symbol.npanels else 0)
