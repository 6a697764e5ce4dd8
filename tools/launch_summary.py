"""Summarise an ncu launch list (gpu__time_duration.sum per launch) by kernel.

    python tools/launch_summary.py gpurun_out/launches.csv [header line]
"""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
h = rows[0]
agg = defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    d = dict(zip(h, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"].split("(")[0]
    agg[name][0] += 1
    agg[name][1] += float(d["Metric Value"]) / 1e3
tot = sum(v[1] for v in agg.values())
if len(sys.argv) > 2:
    print(sys.argv[2])
print("# (cold-cache, serialised replay: compare SHARES, not absolutes)")
print(f"{'kernel':40s} {'launches':>8s} {'total_us':>12s} {'avg_us':>10s} {'share':>6s}")
for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k[:40]:40s} {n:8d} {us:12.1f} {us / n:10.1f} {100 * us / tot:5.1f}%")
