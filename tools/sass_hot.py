"""Hot regions of a kernel from `ncu --page source --csv --print-source sass`:
prints each SASS instruction with executed count and stall samples; with
--blocks, aggregates contiguous address ranges between branch targets."""
import csv, sys

rows = list(csv.reader(open(sys.argv[1])))
# a multi-kernel export repeats (kernel name, header) blocks: keep the first kernel
hdr = rows[1]
for k in range(2, len(rows)):
    if rows[k] and rows[k][0] == "Kernel Name":
        rows = rows[:k]
        break
ia, isrc, isamp, iexe = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
data = [(int(r[ia], 16), r[isrc].strip(), int(r[isamp] or 0), int(r[iexe] or 0)) for r in rows[2:] if len(r) > iexe]
base = data[0][0]
tot_s = sum(d[2] for d in data) or 1
tot_e = sum(d[3] for d in data) or 1
lo = int(sys.argv[2], 16) if len(sys.argv) > 2 else 0
hi = int(sys.argv[3], 16) if len(sys.argv) > 3 else 1 << 40
print(f"total samples {tot_s}, executed {tot_e}")
for a, s, smp, exe in data:
    off = a - base
    if lo <= off <= hi and (exe or smp):
        print(f"{off:05x} {exe:10d} {smp:6d} {100 * smp / tot_s:5.1f}%  {s}")
