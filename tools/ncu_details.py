"""Key 'details' metrics per profiled kernel launch: python tools/ncu_details.py REPORT"""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Executed Ipc Active", "Issued Warp Per Scheduler",
        "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction", "Registers Per Thread",
        "Block Limit Registers", "Block Limit Shared Mem", "Theoretical Occupancy", "Achieved Occupancy",
        "L2 Hit Rate", "L1/TEX Hit Rate", "Issued Instructions", "Avg. Active Threads Per Warp"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
ki, ii, mi, ui, vi = (h.index("Kernel Name"), h.index("ID"), h.index("Metric Name"), h.index("Metric Unit"),
                      h.index("Metric Value"))
cur = None
for r in rows[1:]:
    if len(r) <= vi:
        continue
    if (r[ii], r[ki]) != cur:
        cur = (r[ii], r[ki])
        print(f"== launch {r[ii]} {r[ki][:60]}")
    if r[mi] in KEYS:
        print(f"   {r[mi]:40s} {r[vi]:>14s} {r[ui]}")
