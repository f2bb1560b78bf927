"""Summarise a job directory: pytest tail, bench lines (ms per step, stage times), ncu launch CSVs."""
import csv, glob, json, os, sys
d = sys.argv[1]
p = os.path.join(d, "pytest.txt")
if os.path.exists(p):
    print(open(p).read().strip().splitlines()[-1])
for f in sorted(glob.glob(os.path.join(d, "launches_*.csv"))):
    rows = [r for r in csv.reader(l for l in open(f) if not l.startswith("=="))]
    if not rows: continue
    h = rows[0]; acc = {}
    for r in rows[1:]:
        x = dict(zip(h, r)); acc.setdefault((x["ID"], x["Kernel Name"][:34]), {})[x["Metric Name"]] = x["Metric Value"]
    print("==", os.path.basename(f))
    for (i, k), m in acc.items():
        t = float(m.get("gpu__time_duration.sum", 0)) / 1e3; b = float(m.get("dram__bytes_read.sum", 0))
        print(f"  {k:36s} {t:8.1f} us  {b/1e6:8.1f} MB  {b/1e3/max(t,1e-9)/1e3:6.2f} TB/s  ncu {m.get('dram__throughput.avg.pct_of_peak_sustained_elapsed','')}%")
for f in sorted(glob.glob(os.path.join(d, "bench_*.json"))):
    for l in open(f):
        if l.startswith("{"):
            x = json.loads(l); print(os.path.basename(f), round(x["ms_per_step"], 4), x["roofline"].get("stage_ms"))
