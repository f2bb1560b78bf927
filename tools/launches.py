"""Summarise an ncu --csv launch list (gpu__time_duration.sum per kernel) by kernel name."""
import collections
import csv
import sys


def summarize(path, top=30):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.OrderedDict()
    tot = 0.0
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0]
        v = float(r[vi].replace(",", ""))
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6}[r[ui]]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
        tot += v
    out = [f"total {tot:.1f} us over {sum(c for c, _ in agg.values())} launches"]
    for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        out.append(f"{v:12.1f} us {100 * v / tot:6.2f}%  {c:6d}x  {k[:90]}")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarize(sys.argv[1]))
