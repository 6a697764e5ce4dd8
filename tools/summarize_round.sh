#!/bin/bash
# Copy one round's measurement set (tools/profile_round.sh under gpurun, plus the
# configs[2] sweep launch list and the single-solve latencies) from gpurun_out/ into
# profiles/ with the summaries DESIGN.md cites:  bash tools/summarize_round.sh r02
set -e
tag=${1:-r02}
cd "$(dirname "$0")/.."
grep '^{' gpurun_out/${tag}_bench.log | tail -1 > profiles/${tag}_bench_n1.json
grep '^{' gpurun_out/${tag}_bench_reference.log | tail -1 > profiles/${tag}_bench_reference.json
cp gpurun_out/${tag}_launches.csv profiles/${tag}_launches.csv
python tools/launch_summary.py gpurun_out/${tag}_launches.csv > profiles/${tag}_launches_summary.txt
if [ -f gpurun_out/${tag}_sweep_launches.csv ]; then
  python tools/launch_summary.py gpurun_out/${tag}_sweep_launches.csv \
    "# configs[2] sweep (64 SLO points, max_demand_grid x5 after warm-up; ncu --metrics gpu__time_duration.sum, cold and serialised: compare SHARES)" \
    > profiles/${tag}_sweep_launches_summary.txt
fi
{
  echo "# ncu --set full --clock-control none --import-source on -k regex:'k_s2_exh|k_s1_job|k_x_live|k_m_rank' -s 12 -c 4 python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline (tools/profile_round.sh ${tag}; summarised by tools/ncu_summary.py)"
  python tools/ncu_summary.py gpurun_out/${tag}_full.ncu-rep
} > profiles/${tag}_ncu_full_summary.txt
python tools/ncu_traffic.py gpurun_out/${tag}_full.ncu-rep "profiles/${tag}_ncu_full_summary.txt" > /dev/null
[ -f gpurun_out/${tag}_single.log ] && cp gpurun_out/${tag}_single.log profiles/${tag}_single_solve.txt
echo "profiles/${tag}_* written"
