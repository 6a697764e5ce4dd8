"""Per-instruction view of an ncu source page (SASS): hot instructions and region sums.

usage: python tools/sass_regions.py report.ncu-rep [min_exec] [lo hi]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(out.splitlines()))
h, data = rows[1], rows[2:]
iS = h.index("Warp Stall Sampling (All Samples)")
iE = h.index("Instructions Executed")
tot_s = sum(int(r[iS]) for r in data)
tot_e = sum(int(r[iE]) for r in data)
print("kernel", rows[0][1], "samples", tot_s, "warp-instructions", tot_e, "sass lines", len(data))
mn = int(sys.argv[2]) if len(sys.argv) > 2 else 0
lo = int(sys.argv[3]) if len(sys.argv) > 3 else 0
hi = int(sys.argv[4]) if len(sys.argv) > 4 else len(data)
if mn == 0:
    for k in range(0, len(data), 50):
        seg = data[k:k + 50]
        s = sum(int(r[iS]) for r in seg)
        e = sum(int(r[iE]) for r in seg)
        if s > 0.01 * tot_s or e > 0.01 * tot_e:
            print(f"{k:5d} samples {s / tot_s:.3f} inst {e / tot_e:.3f}")
else:
    for k in range(lo, hi):
        r = data[k]
        if int(r[iE]) >= mn or int(r[iS]) > 0.002 * tot_s:
            print(k, r[1][:64].ljust(64), r[iS].rjust(6), r[iE].rjust(10))
