"""Key numbers of an ncu --set full report (details page).
usage: python tools/ncu_summary2.py REP [REP...]"""
import csv
import subprocess
import sys

WANT = ("Duration", "Executed Ipc Active", "Achieved Occupancy", "Theoretical Occupancy", "DRAM Throughput",
        "Memory Throughput", "Registers Per Thread", "Warp Cycles Per Issued Instruction", "L2 Hit Rate",
        "Shared Memory Configuration Size", "Dynamic Shared Memory Per Block", "Issue Slots Busy")
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    print(f"== {rep}")
    seen = set()
    for r in rows[1:]:
        if len(r) > 14 and r[12] in WANT and (r[4], r[12], r[13]) not in seen:
            seen.add((r[4], r[12], r[13]))
            print(f"  {r[4][:40]:40s} {r[12]:36s} {r[14]:>10s} {r[13]}")
