"""Brief per-kernel ncu metrics from a .ncu-rep: python tools/ncu_brief.py REP [more metric names...]"""
import csv
import io
import subprocess
import sys

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Achieved Occupancy",
        "Registers Per Thread", "Issue Slots Busy", "L2 Hit Rate", "Executed Ipc Active", "Block Limit Registers",
        "Theoretical Occupancy"] + sys.argv[2:]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
for row in rows[1:]:
    d = dict(zip(h, row))
    if d.get("Metric Name") in WANT:
        print(d["ID"], d["Kernel Name"][:60], "|", d["Metric Name"], d["Metric Value"], d["Metric Unit"])
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv", "--metrics",
                      "dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,"
                      "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,"
                      "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"],
                     capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
if rr:
    hh = rr[0]
    idx = [i for i, n in enumerate(hh) if n.startswith(("dram__", "sm__")) or n in ("ID", "Kernel Name")]
    for row in rr[2:]:
        print(" ".join(f"{hh[i]}={row[i][:50]}" for i in idx))
