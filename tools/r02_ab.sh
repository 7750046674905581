#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python bench.py --help > /dev/null
python - <<'PY'
import sys; sys.path.insert(0, ".")
import bench, pathlib
bench._gen_store(pathlib.Path("/tmp"), 10, 0)
PY
SD=/tmp/lubm10
for poll in 1 0; do for into in 1 0; do
  GSM_BATCH_POLL=$poll GSM_BATCH_INTO=$into python tools/e2e_ab.py --reps 400 ${SD:+--store $SD}
done; done | tee gpurun_out/e2e_ab.jsonl
for poll in 1 0; do for into in 1 0; do
  GSM_BATCH_POLL=$poll GSM_BATCH_INTO=$into python tools/e2e_ab.py --reps 400 ${SD:+--store $SD}
done; done | tee -a gpurun_out/e2e_ab.jsonl
python tools/scale_run.py --kind powerlaw --triples 100000000 --node-skew 0.9 --qdir powerlaw_skew \
    --store /tmp/skew100m --only hub_anchored_triangle --reps 5 > gpurun_out/skew_tri.jsonl 2>&1
GSM_NO_INTERSECT=1 python tools/scale_run.py --kind powerlaw --triples 100000000 --node-skew 0.9 \
    --qdir powerlaw_skew --store /tmp/skew100m --only hub_anchored_triangle --reps 5 >> gpurun_out/skew_tri.jsonl 2>&1
grep hub_anchored gpurun_out/skew_tri.jsonl | cut -c1-400
