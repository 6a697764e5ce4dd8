"""profiles/ncu_traffic.json from one ncu --set full capture (per kernel, first launch):
DRAM bytes read/written and issue-slot utilisation, read by bench.py's roofline blocks.

usage: python tools/ncu_traffic.py report.ncu-rep [source-note]"""
import csv
import json
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                     check=True).stdout
rows = list(csv.reader(out.splitlines()))
h, u = rows[0], rows[1]
doc = {"source": (sys.argv[2] if len(sys.argv) > 2 else rep) +
       ": dram__bytes_read.sum + dram__bytes_write.sum and smsp__issue_active, one ncu --set full "
       "capture of bench.py (64 XR solves per launch)"}


def val(d, k):
    v = float(d[k].replace(",", ""))
    unit = u[h.index(k)]
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


for r in rows[2:]:
    d = dict(zip(h, r))
    name = d.get("Kernel Name", "?").split("(")[0].replace("void ", "").split("<")[0].strip()
    if name in doc:
        continue
    doc[name] = {"dram_read_bytes": round(val(d, "dram__bytes_read.sum")),
                 "dram_write_bytes": round(val(d, "dram__bytes_write.sum")),
                 "issue_active_pct": float(d["smsp__issue_active.avg.pct_of_peak_sustained_active"]),
                 "inst_executed": float(d["smsp__inst_executed.sum"].replace(",", "")),
                 "duration_us": val(d, "gpu__time_duration.sum") / (1e3 if u[h.index("gpu__time_duration.sum")] == "ns" else 1)}
json.dump(doc, open("profiles/ncu_traffic.json", "w"), indent=1)
print(json.dumps(doc, indent=1))
