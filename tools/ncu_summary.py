"""Print key ncu --set full metrics per kernel from a .ncu-rep (via ncu -i --page details)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
ki, mi, vi, ui, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
want = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
        "Achieved Occupancy", "Theoretical Occupancy", "Warp Cycles Per Issued Instruction", "No Eligible",
        "Dynamic Shared Memory Per Block", "Block Limit Registers", "Waves Per SM"]
seen = set()
for r in rows[1:]:
    if r[mi] in want and (r[ii], r[mi]) not in seen:
        seen.add((r[ii], r[mi]))
        print(r[ii], r[ki].split("(")[0], "|", r[mi], r[vi], r[ui])
