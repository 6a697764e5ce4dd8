#!/bin/bash
# The round's measurement set (run under gpurun):  bash tools/profile_round.sh r02
#   (then here: bash tools/summarize_round.sh r02 -> profiles/)
#   bench JSON (N=1) and the reference arm; the per-launch list of one bench run
#   (ncu gpu__time_duration, cold and serialised: compare SHARES); one
#   ncu --set full capture of the step's top kernels (k_s2_exh, k_s1_job, k_x_live,
#   k_m_rank) with source correlation.
tag=${1:-r02}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/${tag}_bench.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/${tag}_bench_reference.log 2>&1; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/${tag}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/${tag}_launch_run.log 2>&1
echo "launch list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:'k_s2_exh|k_s1_job|k_x_live|k_m_rank' -s 12 -c 4 -o gpurun_out/${tag}_full \
  python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/${tag}_full_run.log 2>&1
echo "ncu full rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/${tag}_sweep_launches.csv python tools/sweep_run.py > gpurun_out/${tag}_sweep_launch_run.log 2>&1
echo "sweep launch list rc=$?"
timeout 300 python tools/single_latency.py > gpurun_out/${tag}_single.log 2>&1; echo "single rc=$?"
