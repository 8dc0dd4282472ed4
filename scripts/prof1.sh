#!/bin/bash
# ncu --set full of one kernel (regex $1) on the 8192^2 d=0.5 image, library $2 (optional)
cd "$(dirname "$0")/.."
[ -n "$2" ] && export CCL_LIB_PATH=$2
ncu --set full --clock-control none --import-source on -k regex:"$1" -s 2 -c 1 -o gpurun_out/prof1 python scripts/one.py 8192 > gpurun_out/prof1.log 2>&1
