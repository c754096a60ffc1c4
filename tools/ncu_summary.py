"""Summarise an ncu launch list (gpu__time_duration.sum per launch) by kernel.

  python tools/ncu_summary.py gpurun_out/launches_ncu.csv [reps]
The launch list comes from tools/ncu_one.py (reps factorizations after the
plan build); only the last factorization's launches are summarised (the
launches after the last k_assemble)."""
import csv
import collections
import sys

rows = []
with open(sys.argv[1]) as fh:
    lines = [l for l in fh if l.startswith('"')]
for r in csv.DictReader(lines):
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    rows.append((r["Kernel Name"].split("(")[0], float(r["Metric Value"]) / 1e3))
last = max((i for i, (k, _) in enumerate(rows) if k.endswith("assemble")), default=0)
rows = rows[last:]
tot = sum(t for _, t in rows)
by = collections.defaultdict(lambda: [0, 0.0])
for k, t in rows:
    by[k][0] += 1
    by[k][1] += t
print(f"one factorization (assembly + factor), ncu serialised cold-cache: {len(rows)} launches, {tot/1e3:.3f} ms")
print(f"{'kernel':40s} {'launches':>8s} {'ms':>9s} {'share':>7s} {'mean us':>9s}")
for k, (n, t) in sorted(by.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:40s} {n:8d} {t/1e3:9.3f} {t/tot:7.1%} {t/n:9.1f}")
