"""Print an ncu --metrics gpu__time_duration.sum launch list (csv) compactly."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
tot = 0
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        v = float(d["Metric Value"])
        tot += v
        print(f'{d["ID"]:>4} {d["Kernel Name"][:48]:48} grid={d["Grid Size"]:>14} {v/1000:9.2f} us')
print(f"total {tot/1000:.1f} us")
