#!/bin/bash
# compute-sanitizer over every kernel of the labeler (scripts/sanitize_run.py).
# Logs: gpurun_out/sanitize_<tool>.log (summaries copied to profiles/).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
run() {  # name, env, sanitizer args..., -- script args
  local name=$1 envs=$2; shift 2
  env $envs timeout 1500 $CS "$@" > gpurun_out/sanitize_$name.log 2>&1
  echo "$name rc=$?" | tee -a gpurun_out/sanitize_$name.log
  grep -E "SUMMARY|SANITIZE_RUN_DONE" gpurun_out/sanitize_$name.log | tail -3
}
run memcheck "" --tool memcheck --leak-check full --print-limit 200 python scripts/sanitize_run.py
run synccheck "" --tool synccheck --print-limit 200 python scripts/sanitize_run.py
run racecheck "" --tool racecheck --racecheck-report all --print-limit 200 python scripts/sanitize_run.py
# every hazard of a small run listed, for the classification in profiles/
run racecheck_small "" --tool racecheck --racecheck-report all --print-limit 1000000 python scripts/sanitize_run.py small
run initcheck "" --tool initcheck --print-limit 50 python scripts/sanitize_run.py
# initcheck does not track bulk-tensor (TMA) stores as initialising writes:
# the same workload on the generic load/store paths
run initcheck_notma "CCL_NO_TMA=1" --tool initcheck --print-limit 50 python scripts/sanitize_run.py
