#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python - <<'PY'
import sys, pathlib; sys.path.insert(0, ".")
import bench
bench._gen_store(pathlib.Path("/tmp"), 10, 0)
PY
for conn in 8 32 8 32; do
  CUDA_DEVICE_MAX_CONNECTIONS=$conn python tools/e2e_ab.py --reps 400 --store /tmp/lubm10
done | tee gpurun_out/conn_ab.jsonl
CUDA_DEVICE_MAX_CONNECTIONS=32 python tools/batch_probe.py > gpurun_out/batch_probe_conn32.json 2>&1; cat gpurun_out/batch_probe_conn32.json
