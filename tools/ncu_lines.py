"""Per-source-line totals of an ncu source page (SASS csv) for one kernel,
using nvdisasm -g line info of the same cubin.
usage: python tools/ncu_lines.py SASS_CSV ALL_SASS_FROM_NVDISASM KERNEL_SUBSTR [TOP]"""
import csv
import re
import sys
from collections import defaultdict

csv_path, sass_path, kname = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
# offset -> (file, line) for the kernel
lines = open(sass_path).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith(".text.") and kname in l)
off2src = {}
cur = None
for l in lines[start + 1:]:
    if l.startswith(".text.") or l.startswith("//---"):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if m and cur:
        off2src[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(csv_path)))
hdr, data = rows[1], rows[2:]
ie, ss, ad = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Address")
base = min(int(r[ad], 16) for r in data)
agg = defaultdict(lambda: [0.0, 0.0])
for r in data:
    src = off2src.get(int(r[ad], 16) - base, ("?", 0))
    agg[src][0] += float(r[ie] or 0)
    agg[src][1] += float(r[ss] or 0)
ti = sum(v[0] for v in agg.values())
ts = sum(v[1] for v in agg.values())
print(f"total instructions {ti:.3g}, stall samples {ts:.0f}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{k[0]}:{k[1]:<6} inst {v[0]:>11.0f} ({100 * v[0] / ti:4.1f}%)  samples {v[1]:>7.0f} ({100 * v[1] / ts:4.1f}%)")
