#!/bin/bash
# Round artefacts on one GPU: bench line (both arms), ncu launch list of the
# bench command, one ncu --set full capture per kernel.  Outputs under gpurun_out/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_(local|seams|resolve|final)' --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-configs > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k_local|k_seams|k_resolve|k_final' -s 8 -c 4 \
    -o gpurun_out/full python scripts/one.py 8192 > gpurun_out/full.log 2>&1
# summarise locally afterwards: python scripts/summarize_profiles.py r2 gpurun_out/launches.csv gpurun_out/full.ncu-rep
ls -la gpurun_out/full.ncu-rep gpurun_out/launches.csv
