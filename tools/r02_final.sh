#!/usr/bin/env bash
# Round-2 closing measurements: smoke, profiling pass, full bench line and
# the reference arm (what the driver runs), all on one box.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
bash tools/r02_profile.sh > gpurun_out/profile.log 2>&1; tail -5 gpurun_out/profile.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench_rc=$?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench.json").read().strip().splitlines()[-1])
print({k: d[k] for k in ("value", "ms_per_step", "e2e", "roofline", "latency_ms")})
print("scale parity", d["scale_lubm"]["parity"]["ok"], "/", d["scale_lubm"]["parity"]["checked"])
PY
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref_rc=$?"
tail -c 600 gpurun_out/bench_ref.json
