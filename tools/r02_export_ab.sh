#!/usr/bin/env bash
# A/B of the self-cleaning export (loads issued together) against the
# previous build (libgsmat_b200_base.so): LUBM-10 per-query and batch device time.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B=paper_1807_07691_b200/_lib/libgsmat_b200_base.so
N=paper_1807_07691_b200/_lib/libgsmat_b200.so
for lib in $B $N $B $N $B $N; do
  GSM_LIB=$PWD/$lib timeout 300 python tools/l2_probe.py --label "$(basename $lib)" >> gpurun_out/export_ab.jsonl 2>> gpurun_out/export_ab.err
done
python - <<'PY'
import json
for l in open("gpurun_out/export_ab.jsonl"):
    r = json.loads(l)
    c, w = r["cold"], r["warm"]
    print(f'{r["label"]:28s} batch cold {c["batch"]} warm {w["batch"]} | q01 {c["q01"]} q03 {c["q03"]} q10 {c["q10"]} q09 {c["q09"]} | sum cold {round(sum(v for k, v in c.items() if k != "batch"), 4)}')
PY
python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "variants or batch or golden" 2>&1 | tail -2
