#!/usr/bin/env bash
# A/B of the zero-copy limit of fused-projection results (GSM_ZC_BYTES).
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for z in ${ZLIST:-16384 131072 524288 16384 131072 524288}; do
  GSM_ZC_BYTES=$z timeout 300 python tools/l2_probe.py --reps 40 --label "zc=$z" >> gpurun_out/zc_ab.jsonl 2>> gpurun_out/zc_ab.err
done
python - <<'PY'
import json
for l in open("gpurun_out/zc_ab.jsonl"):
    r = json.loads(l)
    c = r["cold"]
    print(r["label"], "batch cold", c["batch"], "warm", r["warm"]["batch"], "q08", c["q08"], "q02", c["q02"], "q04", c["q04"])
PY
