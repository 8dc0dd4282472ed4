set -x
ncu --set full --clock-control none --import-source on -k regex:'k_local|k_final|k_seams' -s 3 -c 3 -o gpurun_out/prof python scripts/one.py 8192 > gpurun_out/prof.log 2>&1
