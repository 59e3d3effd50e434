"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0]
    name = name.replace("void ", "")[:70]
    v = float(r[vi].replace(",", "")) / 1000.0
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(v[1] for v in agg.values())
for k, (n, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:70s} n={n:3d} total={v:9.1f} us  mean={v/n:8.1f} us  {100*v/tot:5.1f}%")
print(f"total {tot:.1f} us")
