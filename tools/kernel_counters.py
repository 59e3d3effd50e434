"""Per-kernel ncu counter table for one bench frame (and optionally one
training view): time, achieved DRAM GB/s and % of the measured HBM peak,
SM / issue / LSU / shared-memory pipe utilisation.

  ncu --metrics $(python tools/kernel_counters.py --metrics) --clock-control none \
      --cache-control none --csv --log-file out.csv python bench.py --no-train --steps 1 --warmup 3
  python tools/kernel_counters.py out.csv > profiles/rNN_kernel_counters.md
"""
import csv
import json
import os
import sys
from collections import OrderedDict

METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
]

if len(sys.argv) > 1 and sys.argv[1] == "--metrics":
    print(",".join(METRICS))
    sys.exit(0)

root = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
peak = 6548.8
try:
    with open(os.path.join(root, "MEASURED_PEAKS.json")) as f:
        mp = json.load(f)
    for k, v in mp.items():
        if "hbm" in k.lower() and isinstance(v, (int, float)):
            peak = float(v)
            break
except Exception:
    pass

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
iid = h.index("ID")
launches = OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    key = r[iid]
    d = launches.setdefault(key, {"name": r[ki].split("(")[0].replace("void ", "")})
    v = float(r[vi].replace(",", ""))
    unit = r[ui]
    if r[mi].startswith("dram__bytes") or r[mi].startswith("lts__t_bytes"):
        v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1)
    if r[mi] == "gpu__time_duration.sum":
        v *= {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}.get(unit, 1.0)
    d[r[mi]] = v
agg = OrderedDict()
for d in launches.values():
    a = agg.setdefault(d["name"], [])
    a.append(d)
print(f"| kernel | launches | mean us | DRAM GB/s | % HBM peak ({peak:.0f}) | L2 GB/s | SM % | issue % | warps % | LSU % | smem % | fp64 % |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|")
for name, ds in sorted(agg.items(), key=lambda kv: -sum(x.get("gpu__time_duration.sum", 0) for x in kv[1])):
    n = len(ds)
    m = lambda k: sum(x.get(k, 0.0) for x in ds) / n
    t = m("gpu__time_duration.sum")
    if t <= 0:
        continue
    gbs = (m("dram__bytes_read.sum") + m("dram__bytes_write.sum")) / (t * 1e-6) / 1e9
    l2 = m("lts__t_bytes.sum") / (t * 1e-6) / 1e9
    print(f"| {name[:48]} | {n} | {t:.1f} | {gbs:.0f} | {100 * gbs / peak:.1f} | {l2:.0f} | "
          f"{m('sm__throughput.avg.pct_of_peak_sustained_elapsed'):.0f} | "
          f"{m('smsp__issue_active.avg.pct_of_peak_sustained_active'):.0f} | "
          f"{m('sm__warps_active.avg.pct_of_peak_sustained_active'):.0f} | "
          f"{m('sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active'):.0f} | "
          f"{m('l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed'):.0f} | "
          f"{m('sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active'):.0f} |")
