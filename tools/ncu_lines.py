"""Aggregate an ncu --page source --csv --print-source cuda,sass export by CUDA source line:
warp-stall samples and executed instructions per line (top N)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
agg = {}
fname = "?"
hdr = None
cur = None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        i_s = hdr.index("Warp Stall Sampling (All Samples)")
        i_e = hdr.index("Instructions Executed")
        continue
    if hdr is None or len(r) <= i_e:
        continue
    if r[0]:
        cur = (fname, int(r[0]), r[1].strip()[:90])
        continue
    if cur is None:
        continue
    try:
        s, e = int(r[i_s] or 0), int(r[i_e] or 0)
    except ValueError:
        continue
    a = agg.setdefault(cur, [0, 0])
    a[0] += s
    a[1] += e
ts = sum(v[0] for v in agg.values())
te = sum(v[1] for v in agg.values())
print(f"total stall samples {ts}, warp instructions {te}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{v[0]:7d} {100*v[0]/max(ts,1):5.1f}% {v[1]:9d}  {k[0]}:{k[1]}  {k[2]}")
