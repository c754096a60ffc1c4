#!/bin/bash
# per-level solve profile (dev): fwd/bwd sums of the last solve call, both forward variants
N=${1:-60}
for g in 0; do
  echo "== PS_SOLVE_GATHER=$g"
  PS_SOLVE_PROFILE=0 python tools/solve_time.py $N 2> /tmp/sp_$g.err
  python - "$g" <<'PY'
import sys, re, collections
lines = open(f"/tmp/sp_{sys.argv[1]}.err").read().splitlines()
runs, cur, prev = [], [], None
for l in lines:
    m = re.match(r"\[solve\] (fwd|bwd) level (\d+) panels (\d+): ([\d.]+) ms", l)
    if not m: continue
    d, L, c, t = m.group(1), int(m.group(2)), int(m.group(3)), float(m.group(4))
    if d == "fwd" and prev == "bwd": runs.append(cur); cur = []
    cur.append((d, L, c, t)); prev = d
runs.append(cur)
r = runs[-1]
print("runs", len(runs), "fwd", round(sum(t for d,_,_,t in r if d=="fwd"),2), "bwd", round(sum(t for d,_,_,t in r if d=="bwd"),2))
for d, L, c, t in sorted(r, key=lambda e: -e[3])[:12]: print(d, L, c, t)
import numpy as np
for d in ("fwd", "bwd"):
    t = np.array([e[3] for e in r if e[0] == d])
    print(d, "levels", len(t), "median ms", np.median(t).round(4), "sum excl. level 0", (t.sum() - max(t)).round(2))
PY
done
