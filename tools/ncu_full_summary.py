"""Key metrics of an ncu --set full report (one launch): section / metric / value, for profiles/.
usage: python tools/ncu_full_summary.py report.ncu-rep "header line" [launch_skip]"""
import csv
import io
import subprocess
import sys

KEEP = ("Memory Throughput", "DRAM Throughput", "Duration", "L1/TEX Cache Throughput", "L2 Cache Throughput",
        "Compute (SM) Throughput", "Mem Busy", "Max Bandwidth", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Issued Warp Per Scheduler", "Warp Cycles Per Issued Instruction", "Issue Slots Busy", "Executed Instructions",
        "Grid Size", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy")
rep, head = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv", "--launch-skip", skip, "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
print(head)
print("kernel:", rows[1][ix["Kernel Name"]])
for r in rows[1:]:
    name = r[ix["Metric Name"]]
    if name in KEEP:
        print(f"{r[ix['Section Name']]:30} {name:45} {r[ix['Metric Value']]:>14} {r[ix['Metric Unit']]}")
