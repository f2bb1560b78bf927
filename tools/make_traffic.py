"""profiles/traffic.json from the ncu --set full summaries of an evidence directory
(tools/evidence_job.sh writes one <name>.json per capture via tools/ncu_traffic.py).

usage: python tools/make_traffic.py profiles/r02/evidence_b"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
d = sys.argv[1]
# config -> capture of the kernel its roofline entry names (bench.py: dominant kernel of the dominant stage)
PICK = {"C1": "lu_small_C1", "C2": "band_spike_C2", "C3a": "potf2_C3a", "C3b": "trsm_C3b", "C4": "jacobi_C4",
        "C5": "gemm_C5", "C5f": "sgemm_C5f"}
out = {}
for tag, name in PICK.items():
    p = os.path.join(d, name + ".json")
    if not os.path.exists(p):
        continue
    try:
        x = json.load(open(p))
    except ValueError:
        continue
    if "dram_bytes" not in x:
        continue
    out[tag] = {"kernel": x["kernel"], "dram_bytes": x["dram_bytes"], "duration_s": x.get("gpu__time_duration.sum"),
                "source": f"{os.path.relpath(d, ROOT)}/{name}.json (ncu --set full --clock-control none, one launch, eager mode)"}
json.dump(out, open(os.path.join(ROOT, "profiles", "traffic.json"), "w"), indent=1)
print(json.dumps(out, indent=1))
