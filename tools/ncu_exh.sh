#!/bin/bash
# one ncu --set full capture of the exhaustive kernel (run under gpurun); $1 = report name
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:k_s2_exh -s 3 -c 1 -o gpurun_out/$1 \
  python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/$1.log 2>&1
