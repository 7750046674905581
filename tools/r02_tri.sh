#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "variants or c3 or lubm or layout or powerlaw" > gpurun_out/tri_pytest.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/tri_pytest.log
python tools/pl_time.py --triples 100000000 --only triangle,chain2,chain3,mix3 --reps 5
python tools/batch_probe.py --reps 30 > gpurun_out/batch_probe4.json 2>&1; cat gpurun_out/batch_probe4.json
