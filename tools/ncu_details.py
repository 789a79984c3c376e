"""Key ncu --set full metrics per kernel from a .ncu-rep (ncu -i ... --page details --csv)."""
import csv
import subprocess
import sys

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Achieved Occupancy",
        "Theoretical Occupancy", "Registers Per Thread", "L2 Hit Rate", "L1/TEX Hit Rate", "Executed Ipc Active",
        "Issue Slots Busy", "Block Limit Registers", "Block Limit Shared Mem", "Grid Size", "Block Size"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
cur = None
for r in rows[1:]:
    d = dict(zip(h, r))
    name = d["Kernel Name"].split("(")[0].replace("void ", "")[-40:] + " #" + d["ID"]
    if name != cur:
        print("==", name)
        cur = name
    if d["Metric Name"] in WANT:
        print(f"   {d['Metric Name']:28s} {d['Metric Value']:>12s} {d['Metric Unit']}")
