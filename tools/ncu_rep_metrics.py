"""Key raw metrics of every launch in an ncu --set full report (one block per
launch): duration, DRAM bytes, instructions, issue utilisation, occupancy,
registers, and the top warp-stall reasons (cycles per issued instruction).
usage: python tools/ncu_rep_metrics.py REP [REP...]"""
import csv
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "sm__inst_executed.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "lts__t_sector_hit_rate.pct", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], dict(zip(rows[0], rows[1]))
    ki = h.index("Kernel Name")
    for r in rows[2:]:
        d = dict(zip(h, r))
        print(f"== {rep}: {r[ki][:70]}")
        for k in WANT:
            if k in d:
                print(f"   {d[k]:>16s} {units[k]:14s} {k}")
        st = sorted(((float(v), k) for k, v in d.items()
                     if "issue_stalled" in k and k.endswith("per_issue_active.ratio") and "not_issued" not in k),
                    reverse=True)[:6]
        print("   stall cycles per issued instruction: " +
              ", ".join(f"{k.split('issue_stalled_')[1].split('_per')[0]} {v:.2f}" for v, k in st))
