#!/bin/bash
# Per-launch device times of our kernels (ncu, serialized, cold-ish caches) for one image kind.
cd "$(dirname "$0")/.."
KIND=${1:-random}
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none ${CACHE_CONTROL:+--cache-control $CACHE_CONTROL} -k regex:'k_' --csv \
  --log-file gpurun_out/launches_$KIND.csv python -c "
import sys; sys.path.insert(0,'.')
import numpy as np, torch, paper_1712_09789_b200 as ccl
img = ccl.random_image(8192,8192,0.5,0) if '$KIND'=='random' else np.zeros((8192,8192),np.uint8)
d = torch.from_numpy(img).cuda()
for _ in range(3): ccl.label_device(d, sync=True)
" > /dev/null 2>&1
