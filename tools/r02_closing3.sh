#!/usr/bin/env bash
# Closing validation of the re-entry session: GPU suite, smoke, bench (both
# arms), ncu launch list + full captures, ingest bench.
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
print("roofline", d["roofline"]["frac"], d["roofline"].get("batched_step"))
sl = d["scale_lubm"]
print("scale parity", sl["parity"]["ok"], "/", sl["parity"]["checked"], "total ms", sl["total"]["ms"])
PY
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref_rc=$?"
tail -c 400 gpurun_out/bench_ref.json
GSM_INGEST_TIMING=1 python tools/ingest_bench.py --univ 10 --ref-univ 2 > gpurun_out/ingest.jsonl 2> gpurun_out/ingest.err
cut -c1-300 gpurun_out/ingest.jsonl; tail -1 gpurun_out/ingest.err
bash tools/r02_profile.sh > gpurun_out/profile.log 2>&1; echo "profile_rc=$?"
