#!/usr/bin/env bash
# A/B of the plan-level L2 prefetch branch (GSM_L2_PREFETCH) on LUBM-10 Q1-Q14:
# per-query and batch device time, cold (after an L2 flush) and warm.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for pf in 0 1 0 1; do
  GSM_L2_PREFETCH=$pf timeout 300 python tools/l2_probe.py --label "pf=$pf" >> gpurun_out/l2pf.jsonl 2> gpurun_out/l2pf.err
  echo "pf=$pf rc=$?"
done
python - <<'PY'
import json
rows = [json.loads(l) for l in open("gpurun_out/l2pf.jsonl")]
for r in rows:
    print(r["label"], "cold", r["cold"]["batch"], "warm", r["warm"]["batch"],
          "q01", r["cold"]["q01"], "q09", r["cold"]["q09"], "sum cold", round(sum(v for k, v in r["cold"].items() if k != "batch"), 3))
PY
