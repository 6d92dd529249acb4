"""Summarise an ncu launch list (gpu__time_duration.sum per launch) by kernel."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = defaultdict(list)
for r in rows[hi + 1:]:
    if len(r) > vi:
        agg[r[ki].split("(")[0][-48:]].append(float(r[vi].replace(",", "")) / 1e3)
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{k:48s} n={len(v):4d} mean={sum(v) / len(v):9.2f} us  share={sum(v) / tot * 100:5.1f}%")
