#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
python - <<'PY'
import subprocess
subprocess.run(["oracle/_build/gsmgen", "powerlaw", "--triples", "100000000", "--predicates", "40",
                "--seed", "0", "--out", "/tmp/pl100m"], check=True, stdout=subprocess.DEVNULL)
PY
for v in "" GSM_NO_INTERSECT=1 GSM_NO_FUSION=1 "" GSM_NO_INTERSECT=1; do
  echo "== $v"; env $v python tools/pl_time.py --store /tmp/pl100m --only triangle,chain2,self_chain,hub_chain --reps 7
done
