"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: total us per kernel name."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
div = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
tot, cnt = defaultdict(float), defaultdict(int)
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0][:70]
    tot[name] += float(r[vi].replace(",", "")) / 1e3
    cnt[name] += 1
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v / div:10.1f} us  n={cnt[k]:4d}  {k}")
