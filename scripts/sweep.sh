#!/bin/bash
# Run scripts/probe.py (args: $PROBE_ARGS) once per experiment library in _lib/.
cd "$(dirname "$0")/.."
for lib in paper_1712_09789_b200/_lib/libccl_b200*.so; do
  echo "== $lib"
  CCL_LIB_PATH=$lib timeout 300 python scripts/probe.py $PROBE_ARGS 2>&1 | tail -n +2
done
