"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) by kernel name (dev tool)."""
import csv, sys, collections
rows = list(csv.reader(l for l in open(sys.argv[1]) if not l.startswith("==")))
hdr = rows[0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
gi = hdr.index("Grid Size") if "Grid Size" in hdr else None
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
top = []
for r in rows[1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum": continue
    name = r[ki].split("(")[0]
    t = float(r[vi].replace(",", "")) * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6}.get(r[hdr.index("Metric Unit")], 1)
    a = agg[name]; a[0] += 1; a[1] += t; a[2] = max(a[2], t)
    top.append((t, name, r[gi] if gi is not None else ""))
tot = sum(a[1] for a in agg.values())
print(f"total {tot/1e3:.3f} us-sum -> {tot/1e6:.3f} ms (serialised)")
for n, a in sorted(agg.items(), key=lambda e: -e[1][1]):
    print(f"{n:30s} n={a[0]:6d} sum={a[1]/1e6:9.3f} ms max={a[2]/1e3:9.1f} us")
print("top launches:")
for t, n, g in sorted(top, reverse=True)[:15]: print(f"  {t/1e3:9.1f} us {n} grid {g}")
