#!/usr/bin/env python
"""Benchmark: numeric factorization GFlop/s on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[4] at one GPU, the metric's own
configuration; it fits one B200): LLt of the 3D 7-point Laplacian 120^3
(n = 1,728,000; 1.0625e13 flops by the reference's flop model on the
reference's own symbol, which this package's analysis reproduces exactly),
one factorization per step.  --size 60 gives configs[1], --size 80 --form
ldlt configs[2].

  python bench.py [--gpus N] [--steps K] [--warmup W] [--size 120] [--form llt]
  python bench.py --impl reference ...      # reference CPU path (oracle port)

value   : flops * K / device time of K steps (CUDA events on the launching
          stream); a step = device assembly of A into the 13.2 GB panel slab
          (> L2, so no flush is needed) + the whole factorization (CUDA-graph
          replay of every level's kernels).  Inputs resident in HBM.
e2e     : the same metric through the public API `factorize(an)` + reading
          the factor back (`res.store`), wall clock per call: H2D of A's
          values from pinned memory, assembly, factorization, pivot check,
          D2H of the whole factor slab into pinned memory.
roofline: dominant kernel = k_update (the DMMA sparse_gemm tiles, inter-
          and intra-panel): tile flops (2 ni nj kn, the reference model's full
          h x h convention) / summed per-launch CUDA-event time of its launches
          (one non-graph pass) vs the measured FP64 DMMA peak
          (tools/fp64_peak.cu, profiles/r01_fp64_peak.txt); traffic = ncu
          dram bytes of one captured launch (profiles/traffic.json).
cpu_baseline: oracle (numpy restatement of the reference kernels) on a
          stratified sample of the same symbol (bench_data/, by source-panel
          width class, extrapolated per class), 1 core, rank 0, N=1 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP64_DMMA_PEAK_TFLOPS = 37.1      # measured, profiles/r01_fp64_peak.txt (DMMA.8x8x4 loop)
FP64_DFMA_PEAK_TFLOPS = 33.9      # measured, same file
METRIC = "factorization GFlop/s & % FP64 peak at 1/2/4/8 B200 vs CPU ref; ||Ax-b||/||b||"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--size", type=int, default=120)
    ap.add_argument("--form", default="llt", choices=["llt", "ldlt", "lu"])
    ap.add_argument("--complex", action="store_true",
                    help="complex128 values (LU: the complex convection-diffusion variant)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def build_matrix(size, form, cplx=False):
    from paper_1405_2636_b200 import sparse
    if form == "lu":  # BASELINE configs[3]: nonsymmetric 27-point convection-diffusion
        return sparse.gen_convdiff27(size, complex_shift=1.0 if cplx else None)
    A = sparse.gen_laplacian(3, (size, size, size))
    if form == "ldlt":
        A = sparse.shift_diagonal(A, 0.5)
    return A


def workload_name(size, form, cplx=False):
    if form == "lu":
        return (f"LU {'complex ' if cplx else ''}double of nonsymmetric 3D 27-point "
                f"convection-diffusion {size}^3" + (" (diagonal + 1i)" if cplx else ""))
    if form == "ldlt":
        return f"LDLT shifted (A-0.5I) 3D 7-point Laplacian {size}^3, double"
    return f"LLT 3D 7-point Laplacian {size}^3, double"


# --------------------------------------------------------------------------
# CPU baseline: the oracle (restated reference kernels) on a stratified sample

def sample_path(size, form):
    return os.path.join(ROOT, "bench_data", f"cpu_sample_{size}_{form}.npz")


def physical_cores():
    try:
        import psutil
        return psutil.cpu_count(logical=False) or os.cpu_count() or 1
    except Exception:  # pragma: no cover
        return os.cpu_count() or 1


def cpu_sample(size, form, workers=1):
    """Reference CPU rate (GFlop/s) estimated from the stratified sample of
    this workload's symbol (tools/make_cpu_sample.py; oracle/cpu_sample.py)."""
    path = sample_path(size, form)
    if not os.path.exists(path):
        return None
    from oracle.cpu_sample import run_sample
    r = run_sample(path, workers)
    r["sample"] = (f"stratified by source-panel width ({len(r['classes'])} classes): "
                   f"{r['units']} factor+update units ({r['sampled_flops']:.3e} of "
                   f"{r['total_flops']:.3e} flop, {r['sampled_seconds']:.1f} s of CPU), each "
                   f"class extrapolated by its flops; the estimate is within 15% of a full "
                   f"oracle / reference run at 60^3 (profiles/r02_cpu_calibration.json)")
    return r


# --------------------------------------------------------------------------
# clocks sampler (pynvml) during the timed region

class ClockSampler:
    def __init__(self, index=0, period=0.1):
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.nv = None
        self.period = period
        self._stop = threading.Event()
        self._t = None

    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
        "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
    }

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in self.REASONS.items():
                    if r & bit and k != "gpu_idle":
                        self.reasons.add(k)
            except Exception:
                pass
            self._stop.wait(self.period)

    def __enter__(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        if self._t:
            self._stop.set()
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# --------------------------------------------------------------------------

def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def run_reference(args):
    """The reference's CPU arithmetic (oracle port of kernels.py, numpy /
    OpenBLAS, 1 BLAS thread per process) on the stratified sample of the
    same workload, all physical cores as independent worker processes (an
    upper bound for the reference's own multi-threaded runtime).  Reads
    only bench_data/; no analysis and no native library of this repo."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    cores = physical_cores()
    if not os.path.exists(sample_path(args.size, args.form)):
        print(json.dumps({"impl": "reference", "unavailable":
                          f"no CPU sample for {args.size}^3 {args.form} "
                          f"(python tools/make_cpu_sample.py {args.size} {args.form})"}))
        return 0
    for _ in range(min(1, args.warmup)):
        cpu_sample(args.size, args.form, workers=cores)
    vals, secs, info = [], 0.0, None
    for _ in range(args.steps):
        info = cpu_sample(args.size, args.form, workers=cores)
        vals.append(info["gflops"])
        secs += info["wall_seconds"]
    v = statistics.median(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "GFlop/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": secs / args.steps * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(args.size, args.form, args.complex),
                   "flops_per_factorization": int(info["total_flops"]),
                   "parallelism": f"cpu: {cores} worker processes x 1 BLAS thread "
                                  "(numpy oracle port of the reference kernels)",
                   "per_core_gflops": info["gflops_per_core"],
                   "logical_cpus": os.cpu_count(), "physical_cores": cores},
        "cpu_baseline": {"value": v, "unit": "GFlop/s", "cores": cores, "kind": "port",
                         "sample": info["sample"]},
        "e2e": {"value": v, "unit": "GFlop/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import torch
    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist
        # PS_DIST_BACKEND=gloo + PS_DIST_SAME_DEVICE=1: functional checks of the
        # multi-rank path on a one-GPU box (not a measurement configuration)
        backend = os.environ.get("PS_DIST_BACKEND", "nccl")
        local = 0 if os.environ.get("PS_DIST_SAME_DEVICE") else local
        torch.cuda.set_device(local)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    from paper_1405_2636_b200 import sparse
    from paper_1405_2636_b200.analysis import AnalyzeOptions, analyze
    from paper_1405_2636_b200.flops import block_flops_array
    from paper_1405_2636_b200.pipeline import default_pivot_threshold, factorize, get_engine

    A = build_matrix(args.size, args.form, args.complex)
    t = time.time()
    an = analyze(A, AnalyzeOptions(form=args.form))
    t_an = time.time() - t
    form = args.form
    thr = default_pivot_threshold(an.A_perm)
    stream = torch.cuda.current_stream(dev)
    t = time.time()
    if ws > 1:
        # multi-GPU: subtree partition, fan-in reduce of the top region, top on rank 0
        from paper_1405_2636_b200.distributed import DistributedFactorizer
        dtop = os.environ.get("PS_DIST_TOP", "1") != "0"
        dfz = DistributedFactorizer(an, rank, ws, dev, distribute_top=dtop,
                                    transport=os.environ.get("PS_DIST_TRANSPORT", "p2p"))
        eng = dfz.engine
        store = dfz.store

        def step():
            dfz.assemble(stream=stream)
            dfz.factor(stream=stream)
    else:
        eng = get_engine(an, dev)
        store = eng.new_store(form, an.is_complex)
        dvals = eng.upload_values(an.A_perm, stream=stream)

        def step():
            eng.assemble(store, an.A_perm, dvals, stream=stream, form=form)
            eng.factor(store, form, thr, stream=stream)
    t_plan = time.time() - t
    torch.cuda.synchronize(dev)

    for _ in range(max(3, args.warmup)):
        step()
    eng.check(form, stream=stream)

    def barrier():
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize(dev)

    # ---- timed region (device events, K steps) ----
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index) as clk:
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        barrier()
    ms = e0.elapsed_time(e1)
    if ws > 1:
        dfz.check(stream=stream)
    else:
        eng.check(form, stream=stream)
    if ws > 1:
        tt = torch.tensor([ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        ms = float(tt.item())
    ms_step = ms / args.steps
    # strong scaling: one factorization of the same matrix per step, all ranks together
    value = an.flops * args.steps / (ms / 1e3) / 1e9
    if ws > 1:
        # ---- e2e through the distributed API: every step H2D of this rank's
        # entries of A from pinned host memory, assembly, factorization, pivot
        # check, D2H of the panels final on this rank (its share of the
        # factor); wall clock, max over the ranks ----
        hv = torch.from_numpy(dfz.host_values()).pin_memory()
        ranges = dfz.owned_ranges()
        nown = sum(n for _, n in ranges)
        hout = torch.empty(nown, dtype=store.dtype, pin_memory=True)
        e2e_steps = max(1, min(args.steps, 3))
        barrier()
        t = time.perf_counter()
        for _ in range(e2e_steps):
            with torch.cuda.stream(stream):
                dfz.dvals.copy_(hv, non_blocking=True)
            dfz.assemble(stream=stream)
            dfz.factor(stream=stream)
            dfz.check(stream=stream)
            o = 0
            with torch.cuda.stream(stream):
                for a, n in ranges:
                    hout[o:o + n].copy_(store[a:a + n], non_blocking=True)
                    o += n
            torch.cuda.synchronize(dev)
        t_e2e = (time.perf_counter() - t) * 1e3 / e2e_steps
        tt = torch.tensor([t_e2e], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t_e2e = float(tt.item())
        # (per-step bytes summed over the ranks)
        bb = torch.tensor([hv.numel() * hv.element_size(), nown * hout.element_size()],
                          device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(bb, op=torch.distributed.ReduceOp.SUM)
        e2e_line = {"value": an.flops / (t_e2e / 1e3) / 1e9, "unit": "GFlop/s",
                    "h2d_bytes_per_step": int(bb[0].item()), "d2h_bytes_per_step": int(bb[1].item()),
                    "ms_per_step": t_e2e,
                    "path": "DistributedFactorizer: H2D of each rank's entries of A (pinned), "
                            "assemble, factor, check, D2H of each rank's final panels (wall "
                            "clock, max over ranks)"}
        full = dfz.gather_factor_slab()
        berr = None
        if rank == 0:
            from paper_1405_2636_b200.pipeline import DeviceStore
            from paper_1405_2636_b200.solve import supernodal_solve
            hstore = DeviceStore(an.symbol, full).to_host()
            b = sparse.spmv(A, np.ones(A.n))
            x = supernodal_solve(an.symbol, hstore, b, form, an.perm.perm)
            berr = sparse.backward_error(A, x, b)
        if rank == 0:
            line = {
                "metric": METRIC, "value": value, "unit": "GFlop/s", "n_gpus": ws,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic",
                "config": {"workload": workload_name(args.size, form), "n": A.n,
                           "flops_per_factorization": an.flops,
                           "parallelism": (f"{ws} GPUs: subtree partition; fan-in by owner-side "
                                           "peer reads of the contributing slabs (CUDA IPC / "
                                           "NVLink); top separators distributed (owners factor, "
                                           "destination owners pull the panels they need and "
                                           "update; device-side epoch flags)")
                                          if dfz.transport == "p2p" else
                                          (f"{ws} GPUs: subtree partition + fan-in all-reduce "
                                           "of the top; top separators distributed (owners "
                                           "factor + broadcast per level, destination owners "
                                           "update)") if dfz.distribute_top else
                                          (f"{ws} GPUs: subtree partition + NCCL fan-in "
                                           "reduce of the top; top on rank 0"),
                           "fp64_peak_frac": value / (ws * FP64_DMMA_PEAK_TFLOPS * 1e3),
                           "backward_error": berr, "analyze_s": t_an, "plan_s": t_plan},
                "roofline": None, "cpu_baseline": None, "e2e": e2e_line,
                "gpu_launches": args.steps * (eng.launches_per_factorization + 1),
                "clocks": clk.summary(),
            }
            print(json.dumps(line), flush=True)
        dfz.close()
        torch.distributed.destroy_process_group()
        return 0

    # ---- correctness of the measured factor: backward error (GPU solve) ----
    b = sparse.spmv(A, np.ones(A.n) * (1 + 0.5j if an.is_complex else 1.0))
    perm = torch.from_numpy(np.ascontiguousarray(an.perm.perm, dtype=np.int64)).to(dev)
    xd = torch.empty(A.n, dtype=store.dtype, device=dev)
    xd[perm] = torch.from_numpy(b).to(dev)
    eng.solve(store, xd, form, stream=stream)
    x = xd[perm].cpu().numpy()
    berr = sparse.backward_error(A, x, b)

    # ---- per-launch device time (non-graph pass, events around every launch) ----
    eng.assemble(store, an.A_perm, dvals, stream=stream, form=form)
    tb = eng.factor_timed(store, form, thr, stream=stream, per_launch=True)
    eng.check(form, stream=stream)
    kinds, _lv, _cnt = eng.launch_table()
    lflops, lbytes = eng.launch_work()
    per = tb["per_launch_ms"]
    # dominant kernel: k_update (DMMA sparse_gemm tiles; inter-panel + intra-panel trailing)
    ku = np.isin(kinds, [2, 3])
    # LU: every tile updates the L and the U slab (2x); complex: 4 real flops
    # per multiply-add slot (flops.py).  Every form's update tiles run on DMMA
    # (complex: k_zupdate, four real DMMA products per fragment pair)
    fmul = (2 if form == "lu" else 1) * (4 if an.is_complex else 1)
    peak = FP64_DMMA_PEAK_TFLOPS
    ku_flops = float(lflops[ku].sum()) * fmul
    ku_ms = float(per[ku].sum())
    achieved = ku_flops / (ku_ms / 1e3) / 1e12
    ku_share = ku_ms / float(per.sum())
    traffic = None
    traffic_note = None
    tfile = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tfile):
        try:
            tj = json.load(open(tfile)).get(f"{args.size}_{form}")
            if tj:
                # the captured launch, identified by (level, tiles) in this plan
                m = np.flatnonzero(ku & (_lv == int(tj["level"])) & (_cnt == int(tj["tiles"])))
                if len(m):
                    idx = int(m[0])
                    traffic = tj["dram_read_bytes"] + tj["dram_write_bytes"]
                    traffic_note = (f"ncu dram bytes of the level-{tj['level']} k_update launch "
                                    f"({tj['tiles']} tiles) vs its algorithmic {lbytes[idx]:.4g} B "
                                    f"({traffic / lbytes[idx]:.2f}x: operand re-reads hit L2); "
                                    f"{tj['fp64_tensor_pct_of_peak_elapsed']}% FP64 tensor peak under ncu")
        except Exception:
            traffic = None

    # ---- e2e through the public API (host buffers, pinned) ----
    e2e = None
    if not args.no_e2e:
        for _ in range(2):
            r = factorize(an, device=dev)
            _ = r.store.slab[0]
        barrier()
        t = time.perf_counter()
        for _ in range(args.steps):
            r = factorize(an, device=dev)
            _ = r.store.slab[0]
        barrier()
        dt = time.perf_counter() - t
        if ws > 1:
            tt = torch.tensor([dt], device=dev, dtype=torch.float64)
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            dt = float(tt.item())
        nv = int(len(eng.assembly(an.A_perm)[1]))  # all of A's values go up (upper ones skipped on device)
        esz = store.element_size()
        e2e = {"value": an.flops * args.steps * ws / dt / 1e9, "unit": "GFlop/s",
               "h2d_bytes_per_step": nv * esz, "d2h_bytes_per_step": store.numel() * esz,
               "ms_per_step": dt / args.steps * 1e3,
               "path": "paper_1405_2636_b200.factorize(an) + FactorResult.store "
                       "(wall clock; H2D of A values, device assembly, factor, pivot "
                       "check, D2H of the factor slab)"}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        info = cpu_sample(args.size, form, workers=1)
        if info is not None:
            cpu = {"value": info["gflops"], "unit": "GFlop/s", "cores": 1, "kind": "port",
                   "sample": info["sample"] + "; 1 process, 1 BLAS thread (the reference's "
                             "fastest configuration, BASELINE.md §2)",
                   "physical_cores": physical_cores()}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GFlop/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "c128" if an.is_complex else "f64", "data": "synthetic",
            "config": {"workload": workload_name(args.size, form, args.complex), "n": A.n,
                       "nnz_l": an.symbol.nnz_l, "panels": an.symbol.npanels,
                       "flops_per_factorization": an.flops,
                       "parallelism": "single GPU" if ws == 1 else f"{ws} independent replicas",
                       "l2": "inputs larger than L2 (slab %.0f MB)" % (store.numel() * store.element_size() / 1e6),
                       "step": "device assembly + factorization (CUDA graph)",
                       "fp64_peak_frac": value / (ws * FP64_DMMA_PEAK_TFLOPS * 1e3),
                       "backward_error": berr, "analyze_s": t_an, "plan_s": t_plan},
            "roofline": {"bound": "tensor",
                         "kernel": ("DMMA complex update tiles: k_zupdate (inter- and "
                                    "intra-panel)" if an.is_complex else
                                    "DMMA update tiles: k_update (large launches), k_update8 "
                                    "(8 warps: launches of < 444 tiles or mean K < 64), "
                                    "k_trail8 (intra-panel trailing tiles)"),
                         "achieved": achieved, "peak": peak,
                         "unit": "TFLOP/s", "frac": achieved / peak,
                         "traffic": traffic, "traffic_note": traffic_note,
                         "peak_source": "measured FP64 DMMA loop (profiles/r01_fp64_peak.txt); "
                                        "MEASURED_PEAKS.json has no FP64 figure",
                         "kernel_ms_per_factorization": ku_ms,
                         "kernel_share_of_step": ku_share,
                         "kernel_flops_per_factorization": ku_flops,
                         "launches": int(ku.sum()),
                         "breakdown_ms": {k: v for k, v in tb.items() if k != "per_launch_ms"}},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": args.steps * (eng.launches_per_factorization + 1),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
