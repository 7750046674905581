#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_chunked.py -x -q -p no:cacheprovider > gpurun_out/ck_pytest.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/ck_pytest.log
for i in 1 2; do
  python bench.py --no-cpu-baseline --no-probe --scale-univ 0 > gpurun_out/bab.json 2> gpurun_out/bab.err
  python - <<'PY'
import json
d = json.loads(open("gpurun_out/bab.json").read().strip().splitlines()[-1])
print("dev", d["ms_per_step"], "e2e", d["e2e"]["ms_per_step"], "e2e_median", d["e2e"].get("median_ms_per_step"),
      "seq", d["sequential"]["ms_per_step"], "seq_e2e", d["sequential"]["e2e_ms_per_step"], d["latency_ms"])
PY
done
