"""Median per-kernel duration from an `ncu --metrics gpu__time_duration.sum --csv` launch list."""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
d = defaultdict(list)
for r in rows[hdr + 1:]:
    if len(r) > vi and r[mi] == "gpu__time_duration.sum":
        d[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")) / 1000.0)
for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
    v = sorted(v)
    print(f"{k:28s} n={len(v):5d} median={v[len(v) // 2]:9.2f} us  total={sum(v):10.1f} us")
