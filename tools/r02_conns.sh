#!/usr/bin/env bash
# Batch concurrency vs the number of hardware work queues (CUDA_DEVICE_MAX_CONNECTIONS).
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for n in 8 32 16 8 32; do
  CUDA_DEVICE_MAX_CONNECTIONS=$n timeout 300 python tools/l2_probe.py --label "conns=$n" >> gpurun_out/conns.jsonl 2>> gpurun_out/conns.err
  echo "conns=$n rc=$?"
done
python - <<'PY'
import json
for l in open("gpurun_out/conns.jsonl"):
    r = json.loads(l)
    print(r["label"], "batch cold", r["cold"]["batch"], "warm", r["warm"]["batch"], "q09", r["cold"]["q09"], "q01", r["cold"]["q01"])
PY
