"""Top stall lines of one kernel in an ncu report: ncu_hot.py REP REGEX [N] [sass|cuda]."""
import csv, subprocess, sys
rep, rx = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
view = sys.argv[4] if len(sys.argv) > 4 else "sass"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{rx}", "-c", "1",
                      "--print-source", view], capture_output=True, text=True).stdout
lines = out.splitlines()
i = next(k for k, l in enumerate(lines) if l.startswith('"Address"') or l.startswith('"Line"') or l.startswith('"#'))
r = list(csv.reader(lines[i:]))
h = r[0]
rows = []
for x in r[1:]:
    d = dict(zip(h, x))
    try:
        v = float(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
    except ValueError:
        v = 0
    rows.append((v, d.get("Address", d.get("Line", "")), d.get("Source", "")[:110]))
tot = sum(v for v, _, _ in rows) or 1
print(f"total samples {tot:.0f}")
for v, a, s in sorted(rows, reverse=True)[:n]:
    print(f"{v:7.0f} {100 * v / tot:5.1f}%  {a}  {s}")
