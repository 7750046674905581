#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_chunked.py tests/test_gpu_tables.py -x -q -p no:cacheprovider > gpurun_out/sc_pytest.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/sc_pytest.log
python - <<'PY'
import sys, pathlib; sys.path.insert(0, ".")
import bench
bench._gen_store(pathlib.Path("/tmp"), 10, 0)
PY
for sc in 0 1 0 1; do
  GSM_NO_SELF_CLEAN=$sc python tools/e2e_ab.py --reps 400 --store /tmp/lubm10
done | tee gpurun_out/sc_ab.jsonl
python tools/batch_probe.py > gpurun_out/batch_probe3.json 2>&1; cat gpurun_out/batch_probe3.json
