"""Per-CUDA-source-line totals of an ncu source page (warp stall samples, warp-instructions).

usage: python tools/ncu_lines.py report.ncu-rep [top_n]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(out.splitlines()))
cur, hdr, res = None, None, []
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0] not in ("", "Function Name"):
        try:
            s, e = int(r[4]), int(r[7])
        except ValueError:
            continue
        res.append((cur, int(r[0]), s, e, r[1][:80]))
ts = sum(x[2] for x in res) or 1
te = sum(x[3] for x in res) or 1
print(f"samples {ts} warp-instructions {te}")
for f, ln, s, e, src in sorted(res, key=lambda x: -x[2])[:top]:
    print(f"{f:22s}{ln:5d} samp {100 * s / ts:5.1f}% inst {100 * e / te:5.1f}%  {src}")
