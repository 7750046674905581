#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_chunked.py tests/test_gpu_tables.py -x -q -p no:cacheprovider > gpurun_out/fz_pytest.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/fz_pytest.log
python bench.py --only-probe > gpurun_out/fz_probe.json 2>&1; cat gpurun_out/fz_probe.json | tail -1
bash tools/r02_bench_ab.sh
