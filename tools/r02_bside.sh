#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "variants or lubm or layout" > gpurun_out/bside_pytest.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/bside_pytest.log
python bench.py --no-cpu-baseline --no-probe --steps 5 > gpurun_out/bside_bench.json 2> gpurun_out/bside_bench.err
echo "bench rc=$?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bside_bench.json").read().strip().splitlines()[-1])
sl = d["scale_lubm"]
print("parity", sl["parity"]["ok"], "/", sl["parity"]["checked"], "total ms", sl["total"]["ms"])
for k, v in sl["queries"].items():
    print(k, v["ms"], v.get("parity"), v.get("fused"))
PY
python - <<'PY'
import subprocess, os
if not os.path.exists("/tmp/wd1000/meta"):
    subprocess.run(["oracle/_build/gsmgen", "watdiv", "--scale", "1000", "--seed", "0", "--out", "/tmp/wd1000"],
                   check=True, stdout=subprocess.DEVNULL)
if not os.path.exists("/tmp/pl100m/meta"):
    subprocess.run(["oracle/_build/gsmgen", "powerlaw", "--triples", "100000000", "--predicates", "40",
                    "--seed", "0", "--out", "/tmp/pl100m"], check=True, stdout=subprocess.DEVNULL)
PY
python tools/scale_run.py --kind watdiv --store /tmp/wd1000 --only C1,C3 --reps 5 --skip-oracle-above 0 2>/dev/null | cut -c1-160
python tools/pl_time.py --store /tmp/pl100m --only chain2,chain3,triangle --reps 7
