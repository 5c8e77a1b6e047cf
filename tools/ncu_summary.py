"""Key metrics per profiled kernel from an ncu report (details page) and the top SASS stall lines."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
want = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Cache Throughput", "L1/TEX Cache Throughput",
        "Compute (SM) Throughput", "Executed Ipc Active", "Achieved Occupancy", "Theoretical Occupancy",
        "Registers Per Thread", "Block Size", "Grid Size", "Dynamic Shared Memory Per Block", "L2 Hit Rate",
        "L1/TEX Hit Rate", "Issue Slots Busy", "No Eligible", "Warp Cycles Per Issued Instruction"]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
cur = None
for r in rows[1:]:
    d = dict(zip(h, r))
    key = (d["ID"], d["Kernel Name"][:40])
    if key != cur:
        cur = key
        print(f"--- [{d['ID']}] {d['Kernel Name'][:70]}")
    if d.get("Metric Name") in want:
        print(f"     {d['Metric Name']:36s} {d['Metric Value']:>12s} {d['Metric Unit']}")
