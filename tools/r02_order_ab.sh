#!/usr/bin/env bash
# A/B: batch members captured longest plan first (GSM_BATCH_ORDER=1) vs input order.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for o in 0 1 0 1 0 1; do
  GSM_BATCH_ORDER=$o timeout 300 python tools/l2_probe.py --reps 60 --label "order=$o" >> gpurun_out/order_ab.jsonl 2>> gpurun_out/order_ab.err
done
python - <<'PY'
import json
for l in open("gpurun_out/order_ab.jsonl"):
    r = json.loads(l)
    print(r["label"], "batch cold", r["cold"]["batch"], "warm", r["warm"]["batch"])
PY
GSM_BATCH_ORDER=1 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "batch" 2>&1 | tail -1
