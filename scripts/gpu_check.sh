#!/bin/bash
# One GPU session: GPU tests, default bench line, N=2 functional runs of the
# multi-GPU bench paths on one GPU, sanitizer.  Logs in gpurun_out/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${T:-all}
if [[ $T == *tests* || $T == all ]]; then
  timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
  tail -3 gpurun_out/gpu_tests.log
fi
if [[ $T == *bench* || $T == all ]]; then
  timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
  tail -c 600 gpurun_out/bench.err
fi
if [[ $T == *multi* || $T == all ]]; then
  for wl in strips32768 batch1080; do
    CCL_BENCH_ONE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
      --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --workload $wl \
      > gpurun_out/bench_n2_$wl.json 2> gpurun_out/bench_n2_$wl.err; echo "n2 $wl rc=$?"
    tail -c 400 gpurun_out/bench_n2_$wl.err
  done
fi
if [[ $T == *san* || $T == all ]]; then
  bash scripts/sanitize.sh
fi
