"""Summarise an ncu report (raw page) for the planner kernels: the counters DESIGN.md cites."""

import csv
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed.sum",
    "smsp__inst_executed.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "sm__cycles_elapsed.avg.per_second",
]
STALLS = "smsp__pcsamp_warps_issue_stalled_"


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(h, r))
        print(f"# kernel {d.get('Kernel Name', '?')}")
        for k in KEYS:
            if k in d:
                print(f"{k} = {d[k]} {u[h.index(k)]}")
        st = sorted(((k[len(STALLS):], float(v.replace(',', '') or 0)) for k, v in d.items()
                     if k.startswith(STALLS) and not k.endswith("not_issued")), key=lambda x: -x[1])
        tot = sum(v for _, v in st) or 1.0
        print("stall samples: " + ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in st[:8]))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
