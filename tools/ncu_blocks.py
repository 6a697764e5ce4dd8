"""Scratch: per-basic-block executed-instruction shares from an ncu source page (SASS)."""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
data = [dict(zip(h, r)) for r in rows[2:]]
ex = [int(d['Instructions Executed'] or 0) for d in data]
samp = [int(d.get('Warp Stall Sampling (All Samples)') or 0) for d in data]
tot = sum(ex)
ts = sum(samp) or 1
print('total', tot)
blocks = []
cur = None
for i, e in enumerate(ex):
    if cur and cur[2] == e:
        cur[1] = i
        cur[3] += e
        cur[4] += samp[i]
    else:
        cur = [i, i, e, e, samp[i]]
        blocks.append(cur)
blocks.sort(key=lambda b: -b[3])
for b in blocks[:int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    print(f"instr {b[0]}-{b[1]} ({b[1]-b[0]+1}) x{b[2]} = {b[3]/tot*100:.1f}% instr, "
          f"{b[4]/ts*100:.1f}% samples | {data[b[0]]['Source'][:50]}")
