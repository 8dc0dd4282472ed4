#!/bin/bash
# bench.py (device value only) for every experiment library in _lib/
cd "$(dirname "$0")/.."
for lib in $(ls paper_1712_09789_b200/_lib/libccl_b200*.so | grep -v metrics1); do
  echo "== $lib"; CCL_LIB_PATH=$lib timeout 300 python bench.py --no-cpu-baseline --steps 30 2>&1 | python -c "
import json,sys
try:
    d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels_ms']
    print(round(d['value'],1), 'Gpx/s', round(d['ms_per_step']*1e3,1), 'us/step | a', round(k['local_ms']*1e3,1), 'd', round(k['merge_ms']*1e3,1), 'e', round(k['final_ms']*1e3,1))
except Exception as e: print('failed', e)"
done
