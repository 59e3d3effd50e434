"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
mi = h.index("Metric Name") if "Metric Name" in h else None
agg = OrderedDict()
extra = OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    if mi is not None and r[mi] != "gpu__time_duration.sum":
        extra.setdefault((r[ki].split("(")[0].replace("void ", "")[:70], r[mi]), []).append(float(r[vi].replace(",", "")))
        continue
    name = r[ki].split("(")[0]
    name = name.replace("void ", "")[:70]
    v = float(r[vi].replace(",", "")) / 1000.0
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(v[1] for v in agg.values())
for k, (n, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    if sys.stdout.closed:
        break
    print(f"{k:70s} n={n:3d} total={v:9.1f} us  mean={v/n:8.1f} us  {100*v/tot:5.1f}%")
print(f"total {tot:.1f} us")
for (k, m), vals in extra.items():
    print(f"{k:70s} {m} mean={sum(vals) / len(vals):.2f}")
