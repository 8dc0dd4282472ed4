#!/bin/bash
# ncu --set full of kernels (d) k_seams and (d2) k_resolve on 8192^2 d=0.5; raw + source CSVs
cd "$(dirname "$0")/.."
for k in k_seams k_resolve; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o gpurun_out/prof_$k python scripts/one.py 8192 > gpurun_out/prof_$k.log 2>&1
  ncu -i gpurun_out/prof_$k.ncu-rep --page raw --csv > gpurun_out/prof_${k}_raw.csv 2>/dev/null
  ncu -i gpurun_out/prof_$k.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/prof_${k}_src.csv 2>/dev/null
done
