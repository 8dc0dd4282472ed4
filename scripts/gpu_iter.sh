#!/bin/bash
# One GPU iteration: quick parity sweep on the default lib, phase breakdown (if a
# phases lib exists), probe sweep over every experiment lib.
cd "$(dirname "$0")/.."
timeout 300 python scripts/check.py > gpurun_out/check.log 2>&1
if [ -f paper_1712_09789_b200/_lib/libccl_b200_phases1.so ]; then
  CCL_LIB_PATH=paper_1712_09789_b200/_lib/libccl_b200_phases1.so timeout 120 python scripts/phases.py 8192 random0.5 zeros spiral > gpurun_out/phases.log 2>&1
fi
PROBE_ARGS="${PROBE_ARGS:---quick}" bash scripts/sweep.sh > gpurun_out/sweep.log 2>&1
