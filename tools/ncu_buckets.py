"""Bucket an ncu source page (warp stall samples, warp-instructions) by source-line ranges.

usage: python tools/ncu_buckets.py report.ncu-rep kernel_substring file:lo-hi=name ..."""
import csv
import subprocess
import sys

rep, ksub = sys.argv[1], sys.argv[2]
ranges = []
for spec in sys.argv[3:]:
    loc, name = spec.split("=")
    f, r = loc.split(":")
    lo, hi = r.split("-")
    ranges.append((f, int(lo), int(hi), name))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", ksub], capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(out.splitlines()))
cur, hdr, agg, ts, te = None, None, {}, 0, 0
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0] not in ("", "Function Name"):
        try:
            s, e, ln = int(r[4]), int(r[7]), int(r[0])
        except ValueError:
            continue
        ts += s
        te += e
        name = "other:" + cur
        for f, lo, hi, nm in ranges:
            if cur == f and lo <= ln <= hi:
                name = nm
                break
        a = agg.setdefault(name, [0, 0])
        a[0] += s
        a[1] += e
print(f"samples {ts} warp-instructions {te}")
for k, (s, e) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{k:40s} samp {100 * s / max(ts, 1):5.1f}%  inst {100 * e / max(te, 1):5.1f}%  ({e})")
