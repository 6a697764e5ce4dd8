#!/bin/bash
# compute-sanitizer over one pass of every libjsv kernel family (tools/sanitize_driver.py),
# run under gpurun; logs and a summary go to gpurun_out/ (copied to profiles/ when judged).
#   usage: bash tools/sanitize.sh [tag]
tag=${1:-r02}
mkdir -p gpurun_out
out=gpurun_out/sanitize_${tag}
: > ${out}_summary.txt
run() {  # $1 = tool, $2 = env label, rest = env assignments
  tool=$1; label=$2; shift 2
  log=${out}_${tool}_${label}.log
  env "$@" timeout 1500 compute-sanitizer --tool ${tool} --error-exitcode 99 --print-limit 2000 \
      python tools/sanitize_driver.py > ${log} 2>&1
  rc=$?
  echo "${tool} ${label} rc=${rc} :: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize driver' ${log} | tr '\n' ' ')" \
      >> ${out}_summary.txt
}
run memcheck default
run memcheck legacy_s1 JSV_S1_LEGACY=1
run memcheck noprune_float JSV_NO_PRUNE=1 JSV_NO_FAST=1
run racecheck default
run racecheck legacy_s1 JSV_S1_LEGACY=1
run synccheck default
run synccheck legacy_s1 JSV_S1_LEGACY=1
run initcheck default
cat ${out}_summary.txt
