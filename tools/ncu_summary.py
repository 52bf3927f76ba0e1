"""Key metrics per kernel from an ncu report: python tools/ncu_summary.py rep.ncu-rep."""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
ki, mi, vi, ui, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
want = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Achieved Occupancy",
        "Registers Per Thread", "Issue Slots Busy", "L2 Hit Rate", "Warp Cycles Per Issued Instruction"]
cur = None
for r in rows[1:]:
    if r[mi] in want:
        k = r[ii] + " " + r[ki].split("(")[0].replace("<unnamed>::", "")
        if k != cur:
            print(k)
            cur = k
        print(f"    {r[mi]:38s} {r[vi]:>12s} {r[ui]}")
