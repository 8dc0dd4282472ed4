#!/bin/bash
# probe.py --quick (timings only) for every experiment library in _lib/: 8192^2 d=0.5 and zeros lines
cd "$(dirname "$0")/.."
for lib in $(ls paper_1712_09789_b200/_lib/libccl_b200*.so | grep -v metrics1); do
  echo "== $lib"; CCL_LIB_PATH=$lib timeout 300 python scripts/probe.py --quick 2>&1 | grep -E "^(random 8192 d0.5|random 8192 d0.7|random 8192 d0.9|spiral 8192|stripes 8192) " | grep " c2fl "
done
