"""Device trace of one dataflow factorization (dev tool).

  python tools/df_trace.py [N] [form]
Per task type: count, wait (ticket -> deps met), body, signal time; the
timeline of running/waiting CTAs; writes gpurun_out/df_trace_<N>_<form>.npz."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1405_2636_b200 import sparse, _abi
from paper_1405_2636_b200.analysis import analyze, AnalyzeOptions
from paper_1405_2636_b200.pipeline import get_engine, default_pivot_threshold

N = int(sys.argv[1]) if len(sys.argv) > 1 else 60
form = sys.argv[2] if len(sys.argv) > 2 else "llt"
A = sparse.gen_laplacian(3, (N, N, N))
if form == "ldlt":
    A = sparse.shift_diagonal(A, 0.5)
an = analyze(A, AnalyzeOptions(form=form))
eng = get_engine(an)
thr = default_pivot_threshold(an.A_perm)
store = eng.new_store()
for _ in range(2):
    eng.assemble(store, an.A_perm); eng.factor(store, form, thr); eng.check(form)
eng.assemble(store, an.A_perm)
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); eng.factor(store, form, thr); e1.record(); eng.check(form)
ms = e0.elapsed_time(e1)
eng.assemble(store, an.A_perm)
tr = eng.factor_trace(store, form, thr)
eng.check(form)
ty, src, dst, fl = eng.tasks()
T = tr[:, :4].astype(np.int64)
base = T[:, 0].min()
T = (T - base) / 1e3  # us
tw, ts, tb, te = T[:, 0], T[:, 1], T[:, 2], T[:, 3]
span = te.max()
di = eng.dataflow_info()
G = di["grid"]
print(f"N={N} {form}: graph {ms:.3f} ms ({an.flops/ms/1e9:.2f} TF); traced span {span/1e3:.3f} ms; "
      f"sim est {di['est_ms']:.3f} ms; tasks {len(ty)}; grid {G}")
print(f"  CTA time: waiting {(ts-tw).sum()/1e3:.1f} ms, body {(tb-ts).sum()/1e3:.1f} ms, "
      f"signal {(te-tb).sum()/1e3:.1f} ms of {G*span/1e3:.1f} CTA-ms")
for k, name in enumerate(_abi.DT_NAMES):
    sel = ty == k
    if sel.any():
        b = (tb - ts)[sel]; w = (ts - tw)[sel]; g = (te - tb)[sel]
        print(f"  {name:12s} n {sel.sum():7d}  body {b.sum()/1e3:8.1f} CTA-ms mean {b.mean():6.2f} p50 {np.median(b):6.2f} "
              f"max {b.max():7.1f} us | wait mean {w.mean():7.2f} us | signal mean {g.mean():5.2f} us | "
              f"{fl[sel].sum()/max(b.sum(),1e-9)/1e3:.1f} GF/s/CTA")
nb = 20
edges = np.linspace(0, span, nb + 1)
print("  timeline: CTAs in body / waiting, per bucket")
for b in range(nb):
    lo, hi = edges[b], edges[b + 1]
    body = np.clip(np.minimum(tb, hi) - np.maximum(ts, lo), 0, None)
    wait = np.clip(np.minimum(ts, hi) - np.maximum(tw, lo), 0, None)
    bytype = [body[ty == k].sum() / (hi - lo) for k in range(len(_abi.DT_NAMES))]
    print(f"   {lo/1e3:7.3f}-{hi/1e3:7.3f} ms  body {body.sum()/(hi-lo):6.1f} wait {wait.sum()/(hi-lo):6.1f}  " +
          " ".join(f"{_abi.DT_NAMES[k][:5]}={bytype[k]:.0f}" for k in range(len(bytype)) if bytype[k] >= 0.5))
os.makedirs("gpurun_out", exist_ok=True)
np.savez_compressed(f"gpurun_out/df_trace_{N}_{form}.npz", type=ty, src=src, dst=dst, flops=fl,
                    t=T, sm=(tr[:, 4] >> 8).astype(np.int64))

# ---- measured critical path: walk back from the last task through the
#      dependency that was released last ----
dep_ptr, dep_ctr, dep_tg, sig_ptr, sig_ctr = eng.task_graph()
nt = len(ty)
# release time of (counter, value): the value-th signal event on the counter
ev_ctr = np.repeat(np.arange(nt), np.diff(sig_ptr))
ev_t = te[ev_ctr]
order = np.lexsort((ev_t, sig_ctr))
sc = sig_ctr[order]
first = np.searchsorted(sc, np.arange(sc.max() + 2 if len(sc) else 1))
def releaser(c, v):
    k = first[c] + v - 1
    return ev_ctr[order[k]]
t = int(np.argmax(te))
path = []
while True:
    path.append(t)
    best, bt = -1, -1.0
    for k in range(dep_ptr[t], dep_ptr[t + 1]):
        u = releaser(dep_ctr[k], dep_tg[k])
        if te[u] > bt:
            bt, best = te[u], u
    if best < 0:
        break
    t = best
path = path[::-1]
seg = {"body": 0.0, "signal": 0.0, "ready->start": 0.0}
bytype = {}
for a, b in zip(path[:-1], path[1:]):
    seg["ready->start"] += max(0.0, ts[b] - te[a])
for t in path:
    seg["body"] += tb[t] - ts[t]
    seg["signal"] += te[t] - tb[t]
    nm = _abi.DT_NAMES[ty[t]]
    bytype[nm] = bytype.get(nm, 0.0) + (te[t] - ts[t])
print(f"  critical path: {len(path)} tasks, {(te[path[-1]] - ts[path[0]])/1e3:.3f} ms: "
      + ", ".join(f"{k} {v/1e3:.3f} ms" for k, v in seg.items()))
print("   by type (body+signal): " + ", ".join(f"{k} {v/1e3:.3f} ms" for k, v in sorted(bytype.items(), key=lambda kv: -kv[1])))
pa = np.array(path)
print("   path segments by type: " + ", ".join(
    f"{_abi.DT_NAMES[k]} n={int((ty[pa]==k).sum())} body={((tb-ts)[pa][ty[pa]==k]).sum()/1e3:.2f}ms"
    for k in range(len(_abi.DT_NAMES)) if (ty[pa] == k).any()))
longest = pa[np.argsort(-(tb - ts)[pa])[:12]]
for t in longest:
    print(f"     long path task {t}: {_abi.DT_NAMES[ty[t]]} src {src[t]} dst {dst[t]} body {tb[t]-ts[t]:.1f} us "
          f"signal {te[t]-tb[t]:.1f} us flops {fl[t]:.3g}")
# path timeline: how much of the path lies in each tenth of the run
np.savez_compressed(f"gpurun_out/df_path_{N}_{form}.npz", path=pa)
ph = eng.last_phase.astype(np.int64)
gsel = np.where((ty == 5) & (ph[:, 3] > 0))[0]
if len(gsel):
    P = (ph[gsel] - base) / 1e3
    st = ts[gsel]
    d = np.stack([P[:, 0] - st, P[:, 1] - P[:, 0], P[:, 2] - P[:, 1], P[:, 3] - P[:, 2], tb[gsel] - P[:, 3]], 1)
    print("  gather phases mean us (desc, loads, inv, compute, store):", np.round(d.mean(0), 2))
    slow = np.argsort(-(tb[gsel] - ts[gsel]))[:8]
    for k in slow:
        print("    slow gather", gsel[k], "phases", np.round(d[k], 1))
