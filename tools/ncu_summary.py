"""Key metrics per kernel from an ncu --page details --csv export."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[0]
ii, ki, mi, vi, ui = (h.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
want = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Cache Throughput", "L1/TEX Cache Throughput",
        "Compute (SM) Throughput", "Executed Ipc Active", "Achieved Occupancy", "Theoretical Occupancy",
        "Registers Per Thread", "Warp Cycles Per Issued Instruction", "L2 Hit Rate", "Issued Instructions",
        "Grid Size", "Block Size", "Dynamic Shared Memory Per Block", "Static Shared Memory Per Block"]
seen = {}
for r in rows[1:]:
    if len(r) <= vi or r[mi] not in want:
        continue
    key = (r[ii], r[ki][:60])
    seen.setdefault(key, {})[r[mi]] = f"{r[vi]} {r[ui]}"
for (i, k), d in seen.items():
    print(f"== [{i}] {k}")
    for w in want:
        if w in d:
            print(f"   {w:38s} {d[w]}")
