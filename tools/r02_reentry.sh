#!/usr/bin/env bash
# Re-entry check after a container rebuild: GPU suite, smoke, bench line.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest_rc=$?"; tail -2 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench_rc=$?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench.json").read().strip().splitlines()[-1])
print({k: d[k] for k in ("value", "ms_per_step", "e2e", "latency_ms", "gpu_launches", "clocks")})
print("roofline", d["roofline"]["frac"], d["roofline"]["us_per_step"])
sl = d["scale_lubm"]
print("scale parity", sl["parity"]["ok"], "/", sl["parity"]["checked"], "total ms", sl["total"]["ms"])
PY
