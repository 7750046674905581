#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
start=$(date +%s)
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench_rc=$? wall=$(( $(date +%s) - start ))s"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench.json").read().strip().splitlines()[-1])
print({k: d[k] for k in ("value", "ms_per_step", "e2e", "gpu_launches", "clocks")})
for key in ("scale_lubm", "scale_watdiv"):
    sl = d[key]
    print(key, "parity", sl["parity"]["ok"], "/", sl["parity"]["checked"], "total ms", sl["total"]["ms"])
PY
start=$(date +%s)
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref_rc=$? wall=$(( $(date +%s) - start ))s"
python -c "
import json; d=json.loads(open('gpurun_out/bench_ref.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'])"
