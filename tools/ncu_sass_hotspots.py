"""Per-SASS-instruction hot spots from `ncu -i rep --page source --csv --print-source sass`:
instructions executed and warp-stall sample share, for lines above a threshold."""
import csv, sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
ia, isamp = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
iavg = hdr.index("Avg. Predicated-On Threads Executed")
num = lambda v: int(v) if v.isdigit() else 0
tot = sum(num(r[ia]) for r in data)
ts = sum(num(r[isamp]) for r in data)
print(rows[0][1])
print(f"instructions executed {tot}, stall samples {ts}")
print("addr   inst(M) stall%  thr  sass")
for r in data:
    n, sm = num(r[ia]), num(r[isamp])
    if n > tot * 0.004 or sm > ts * 0.01:
        print(f"{r[0][-5:]} {n/1e6:7.2f} {100*sm/ts:6.1f} {r[iavg]:>4}  {r[1].strip()[:80]}")
