#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
python - <<'PY'
import subprocess, os
if not os.path.exists("/tmp/wd1000/meta"):
    subprocess.run(["oracle/_build/gsmgen", "watdiv", "--scale", "1000", "--seed", "0", "--out", "/tmp/wd1000"],
                   check=True, stdout=subprocess.DEVNULL)
PY
D=$PWD/paper_1807_07691_b200/_lib
for rnd in 1 2; do
for lib in $D/libgsmat_b200_1ce14e5.so $D/libgsmat_b200_3a19084.so $D/libgsmat_b200_cb60626.so $D/libgsmat_b200.so; do
  echo "== $(basename $lib)"
  GSM_LIB=$lib python tools/scale_run.py --kind watdiv --store /tmp/wd1000 --only C1,C3,F3,F4 --reps 5 \
    --skip-oracle-above 0 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if 'query' in d: print(' ', d['query'], d['gpu_ms'])
"
done
done
