"""GPU factorization timelines in the reference's trace schema.

The reference's runtime records one `TraceEvent(task_id, kind, p, q, worker,
start_ns, end_ns)` per task and writes them as CSV
`task_id,kind,src,dst,worker,start_ns,end_ns` (runtime.py:28-36, 325-348).
Here a task is refined into tiles and level-batched launches; its event
spans the launches that work on it (ps_plan_launch_tasks), timed with CUDA
events around every launch (ps_factor_timeline: launches serialized on one
stream, the graph's concurrent branches become the `worker` lanes).
"""

from __future__ import annotations

import csv
from dataclasses import dataclass

import numpy as np

from .taskgraph import FACTOR, UPDATE, couples

TRACE_FIELDS = ["task_id", "kind", "src", "dst", "worker", "start_ns", "end_ns"]


@dataclass
class TraceEvent:
    task_id: int
    kind: str
    p: int
    q: int
    worker: int
    start_ns: int
    end_ns: int


def trace_to_csv(events, path):
    """CSV trace, one row per event, sorted by start (runtime.py:325-336)."""
    rows = sorted(events, key=lambda e: (e.start_ns, e.task_id))
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(TRACE_FIELDS)
        for e in rows:
            w.writerow([e.task_id, e.kind, e.p, e.q, e.worker, e.start_ns, e.end_ns])


def read_trace_csv(path):
    """Inverse of trace_to_csv (runtime.py:339-348)."""
    with open(path, newline="") as fh:
        return [TraceEvent(int(r["task_id"]), r["kind"], int(r["src"]), int(r["dst"]),
                           int(r["worker"]), int(r["start_ns"]), int(r["end_ns"]))
                for r in csv.DictReader(fh)]


def launch_tasks(engine):
    """(ptr[nlaunch + 1], task ids) of every launch (ps_plan_launch_tasks)."""
    from ._native import ptr
    n = int(engine.info["nlaunches"])
    lp = np.zeros(n + 1, dtype=np.int64)
    engine._check(engine.lib.ps_plan_launch_tasks(engine.handle, ptr(lp), None))
    tk = np.zeros(max(1, int(lp[-1])), dtype=np.int64)
    engine._check(engine.lib.ps_plan_launch_tasks(engine.handle, ptr(lp), ptr(tk)))
    return lp, tk[:int(lp[-1])]


def events_from_timeline(symbol, engine, start_ms, dur_ms):
    """One TraceEvent per reference task from per-launch start / duration (ms)."""
    lp, tk = launch_tasks(engine)
    branch = engine.launch_table(branches=True)[3]
    nl = len(lp) - 1
    li = np.repeat(np.arange(nl), np.diff(lp))
    s_ns = np.round(np.asarray(start_ms, dtype=np.float64) * 1e6).astype(np.int64)
    e_ns = s_ns + np.round(np.asarray(dur_ms, dtype=np.float64) * 1e6).astype(np.int64)
    cp, cq, _, _ = couples(symbol)
    ntask = symbol.npanels + len(cp)
    t0 = np.full(ntask, np.iinfo(np.int64).max)
    t1 = np.full(ntask, -1, dtype=np.int64)
    wk = np.zeros(ntask, dtype=np.int64)
    np.minimum.at(t0, tk, s_ns[li])
    np.maximum.at(t1, tk, e_ns[li])
    wk[tk] = branch[li]
    ev = []
    npn = symbol.npanels
    for t in np.flatnonzero(t1 >= 0).tolist():
        if t < npn:
            ev.append(TraceEvent(t, FACTOR, t, t, int(wk[t]), int(t0[t]), int(t1[t])))
        else:
            c = t - npn
            ev.append(TraceEvent(t, UPDATE, int(cp[c]), int(cq[c]), int(wk[t]), int(t0[t]), int(t1[t])))
    ev.sort(key=lambda e: (e.start_ns, e.task_id))
    return ev
