#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
python - <<'PY'
import sys, pathlib; sys.path.insert(0, ".")
import bench
bench._gen_store(pathlib.Path("/tmp"), 10, 0)
PY
for v in 0 1 0 1; do GSM_BATCH_PDL=$v python tools/e2e_ab.py --reps 400 --store /tmp/lubm10; done
GSM_BATCH_PDL=1 python tools/batch_probe.py --reps 30
