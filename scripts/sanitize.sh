#!/bin/bash
# compute-sanitizer over every kernel of the labeler (scripts/sanitize_run.py).
# Logs: gpurun_out/sanitize_<tool>.log (copied to profiles/ by hand).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check full"
  [ "$tool" = racecheck ] && extra="--racecheck-report all"
  timeout 1500 $CS --tool $tool $extra --print-limit 200 python scripts/sanitize_run.py \
    > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/sanitize_$tool.log
  tail -3 gpurun_out/sanitize_$tool.log
done
