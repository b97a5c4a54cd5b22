"""Summarise an `ncu --set full` report into the JSON kept under profiles/
(development aid).  usage: python dev/ncu_summary.py REPORT.ncu-rep "source text" > out.json"""
import csv, io, json, subprocess, sys

KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "smsp__inst_executed.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__cycles_active.avg", "gpc__cycles_elapsed.max",
        "launch__grid_size", "launch__block_size", "launch__cluster_dim_x",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed"]

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(out)))
head, units, data = rows[0], rows[1], rows[2:]
kernels = []
for r in data:
    d = {}
    for k in KEYS:
        if k in head:
            i = head.index(k)
            d[k] = f"{r[i]} {units[i]}".strip() if k != "Kernel Name" else r[i]
    kernels.append(d)
print(json.dumps({"source": sys.argv[2] if len(sys.argv) > 2 else rep, "kernels": kernels}, indent=1))
