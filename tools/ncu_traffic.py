"""DRAM bytes / duration / DMMA activity of the single kernel in an ncu --set full report.

usage: python tools/ncu_traffic.py report.ncu-rep [...]   -> one JSON object per report
"""
import csv
import io
import json
import subprocess
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
         "s": 1.0, "KB": 1e3, "MB": 1e6, "GB": 1e9, "B": 1, "": 1, "%": 1}
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__inst_executed_pipe_fp64.sum", "smsp__inst_executed_pipe_fp64.sum",
           "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
           "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"]


def read(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[-1]
    d = {"kernel": vals[hdr.index("Kernel Name")], "report": path}
    for m in METRICS:
        if m in hdr:
            i = hdr.index(m)
            try:
                d[m] = float(vals[i].replace(",", "")) * SCALE.get(units[i], 1)
            except ValueError:
                pass
    d["dram_bytes"] = d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    return d


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(json.dumps(read(p)))
