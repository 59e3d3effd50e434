"""Print the headline metrics of an ncu report (first kernel): time, DRAM,
pipes, issue, occupancy, stall reasons, opcode mix."""
import csv, io, subprocess, sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, v = rows[0], rows[2]
d = dict(zip(h, v))
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_bytes.sum"]
for k in want:
    if k in d:
        print(f"{k:70s} {d[k]}")
st = []
for k, x in d.items():
    if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
        try:
            st.append((float(x.replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
tot = sum(a for a, _ in st) or 1
print("stalls:", ", ".join(f"{n} {a / tot:.0%}" for a, n in sorted(st, reverse=True)[:9]))
if "sass__inst_executed_per_opcode" in d:
    print("opcodes:", d["sass__inst_executed_per_opcode"][:700])
