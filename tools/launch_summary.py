"""Summarise an ncu --csv launch list (gpu__time_duration.sum [+ dram bytes]): per kernel name."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
div = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
d, ids = defaultdict(lambda: defaultdict(float)), defaultdict(set)
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0][:60]
    d[name][r[mi]] += float(r[vi].replace(",", ""))
    ids[name].add(r[ii])
for k, v in sorted(d.items(), key=lambda x: -x[1]["gpu__time_duration.sum"]):
    t = v["gpu__time_duration.sum"] / 1e3 / div
    rd, wr = v.get("dram__bytes_read.sum", 0) / 1e9 / div, v.get("dram__bytes_write.sum", 0) / 1e9 / div
    bw = (rd + wr) / (t * 1e-6) if t else 0
    print(f"{t:10.1f} us  rd {rd:7.3f} GB  wr {wr:7.3f} GB  {bw:7.0f} GB/s  n={len(ids[k]):4d}  {k}")
