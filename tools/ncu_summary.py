"""Summarise an ncu report: key metrics, top SASS stalls, per-source-line instruction counts."""
import csv, subprocess, sys
rep = sys.argv[1]
kernel_filter = sys.argv[2] if len(sys.argv) > 2 else None
def run(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout
r = list(csv.reader(run("--page", "details", "--csv").splitlines()))
hdr = r[0]
keys = ['Duration', 'DRAM Throughput', 'Memory Throughput', 'Executed Ipc Active', 'Issue Slots Busy',
        'Eligible Warps', 'Warp Cycles Per Issued', 'Executed Instructions', 'Achieved Occupancy',
        'Registers Per', 'L2 Hit Rate', 'Block Limit Registers', 'Grid Size']
for row in r[1:]:
    d = dict(zip(hdr, row))
    n = d.get('Metric Name', '')
    if any(n.startswith(k) for k in keys):
        print(n[:42].ljust(42), d.get('Metric Unit', '')[:10].ljust(10), d.get('Metric Value', ''))
rows = list(csv.reader(run("--page", "source", "--csv", "--print-source", "cuda,sass").splitlines()))
agg, srcline, cur, last = {}, {}, None, None
def f(x):
    try: return float(x)
    except Exception: return 0.0
for row in rows:
    if not row: continue
    if row[0] in ('File Path', 'Function Name', 'Line No'):
        if row[0] == 'File Path': cur = row[1].split('/')[-1]
        continue
    ln = row[0]
    ie, ss = (f(row[7]) if len(row) > 7 else 0), (f(row[4]) if len(row) > 4 else 0)
    if ln:
        last = (cur, ln); srcline[last] = row[1]; agg.setdefault(last, [0, 0])
    if last:
        agg[last][0] += ie; agg[last][1] += ss
tot_i = sum(v[0] for v in agg.values()); tot_s = sum(v[1] for v in agg.values())
print(f"--- per source line (instr share / stall share), totals {tot_i:.3g} / {tot_s:.3g}")
for k, v in sorted(agg.items(), key=lambda kv: -(kv[1][0] / max(tot_i, 1) + kv[1][1] / max(tot_s, 1)))[:int(sys.argv[3]) if len(sys.argv) > 3 else 30]:
    print(k[0][:13].ljust(13), k[1].rjust(5), f"{100*v[0]/max(tot_i,1):5.1f}% {100*v[1]/max(tot_s,1):5.1f}%", srcline[k].strip()[:85])
