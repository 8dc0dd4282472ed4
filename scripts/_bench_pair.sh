cd "$(dirname "$0")/.."
timeout 300 python scripts/check.py > gpurun_out/check.log 2>&1
for lib in paper_1712_09789_b200/_lib/libccl_b200.so paper_1712_09789_b200/_lib/libccl_b200_pdl0.so; do
  echo "== $lib"; CCL_LIB_PATH=$lib timeout 300 python bench.py --no-cpu-baseline --steps 30 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],1), 'Gpx/s', round(d['ms_per_step']*1e3,1), 'us/step', d['kernels_ms'], 'e2e', round(d['e2e']['value'],2))"
done > gpurun_out/benchpair.log 2>&1
