"""Top CUDA source lines by warp-stall samples from an ncu report's source page.

  ncu -i rep.ncu-rep --page source --csv --print-source cuda,sass > src.csv
  python tools/ncu_src_top.py src.csv [N]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname = None
hdr = None
per = []
tot = 0
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 3 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 5 or r[0] in ("", "Function Name"):
        continue
    try:
        samp = int(r[4])
    except ValueError:
        continue
    tot += samp
    stalls = {}
    for k, name in enumerate(hdr):
        if name.startswith("stall_") and "Not Issued" not in name:
            try:
                v = int(r[k])
            except ValueError:
                continue
            if v:
                stalls[name[6:]] = v
    per.append((samp, fname, r[0], r[1][:100], stalls))
per.sort(key=lambda x: -x[0])
print(f"total samples {tot}")
for samp, f, ln, src, st in per[:N]:
    top = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    print(f"{samp/tot:6.1%} {f}:{ln:5s} {src.strip()}")
    if top:
        print("           " + ", ".join(f"{k}={v}" for k, v in top))
