#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in "GSM_BENCH_GC=1" "GSM_BENCH_GC=0" "GSM_BENCH_GC=1" "GSM_BENCH_GC=0"; do
  env $v python bench.py --no-cpu-baseline --no-probe --scale-univ 0 > gpurun_out/bab.json 2> gpurun_out/bab.err
  python - "$v" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/bab.json").read().strip().splitlines()[-1])
print(sys.argv[1] or "default", "dev", d["ms_per_step"], "e2e", d["e2e"]["ms_per_step"],
      "e2e_median", d["e2e"].get("median_ms_per_step"),
      "seq", d["sequential"]["ms_per_step"], "seq_e2e", d["sequential"]["e2e_ms_per_step"])
PY
done
python bench.py --only-probe > gpurun_out/fz_probe.json 2>&1; tail -1 gpurun_out/fz_probe.json
