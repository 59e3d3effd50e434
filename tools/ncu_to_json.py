"""Read the headline metrics of the first kernel of an ncu report into the
JSON bench.py uses for roofline.traffic (profiles/r02_blend_ncu.json).
usage: ncu_to_json.py REPORT.ncu-rep OUT.json "config note" "source note" """
import csv, io, json, subprocess, sys

rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
d = dict(zip(rows[0], rows[2]))
units = dict(zip(rows[0], rows[1]))


def num(k, scale=1.0):
    v = float(d[k].replace(",", ""))
    u = units.get(k, "")
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3}.get(u, 1)
    return v * mult * scale


j = {"kernel": d["Kernel Name"].split("(")[0].replace("void ", ""),
     "config": sys.argv[3] if len(sys.argv) > 3 else "",
     "source": sys.argv[4] if len(sys.argv) > 4 else rep,
     "dram_read_bytes": int(num("dram__bytes_read.sum")), "dram_write_bytes": int(num("dram__bytes_write.sum")),
     "duration_us": num("gpu__time_duration.sum"),
     "issue_active": num("smsp__issue_active.avg.pct_of_peak_sustained_active") / 100,
     "fp64_pipe_active": num("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active") / 100,
     "alu_pipe_active": num("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active") / 100,
     "warps_active": num("sm__warps_active.avg.pct_of_peak_sustained_active") / 100,
     "warp_instructions": int(num("smsp__inst_executed.sum")),
     "registers_per_thread": int(num("launch__registers_per_thread"))}
j["dram_bytes"] = j["dram_read_bytes"] + j["dram_write_bytes"]
json.dump(j, open(out, "w"), indent=1)
print(json.dumps(j))
