"""Per-kernel shares of the first K launches of an ncu --csv launch list
(serialised, cold-cache durations): python tools/step_shares.py launches.csv K STEPS"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
K, steps = int(sys.argv[2]), int(sys.argv[3])
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = defaultdict(dict)
for r in rows[hdr + 1:]:
    if len(r) > vi:
        per[int(r[ii])][r[mi]] = float(r[vi].replace(",", ""))
        per[int(r[ii])]["name"] = r[ki].split("(")[0].replace("void ", "")[:48]
ids = sorted(per)[:K]
tot = defaultdict(float)
for i in ids:
    tot[per[i]["name"]] += per[i]["gpu__time_duration.sum"]
allt = sum(tot.values())
print(f"{K} launches, {allt / 1e6 / steps:.2f} ms per step serialised")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"  {v / allt * 100:5.1f} %  {v / 1e6 / steps:7.2f} ms/step  {k}")
