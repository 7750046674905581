#!/usr/bin/env bash
# Triangle / cyclic queries with and without the fused intersection path
# (GSM_NO_INTERSECT=1), power-law 100M and LUBM-100 complex queries.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TRIPLES:-100000000}
python tools/scale_run.py --kind powerlaw --triples $T --predicates 40 --reps 5 --only triangle,mix3,self_chain,chain2 > gpurun_out/isect_pl.jsonl 2>&1
GSM_NO_INTERSECT=1 python tools/scale_run.py --kind powerlaw --triples $T --predicates 40 --reps 5 --only triangle,mix3,self_chain,chain2 --skip-oracle-above 0 > gpurun_out/isect_pl_off.jsonl 2>&1
python tools/scale_run.py --univ ${UNIV:-100} --reps 5 > gpurun_out/isect_lubm.jsonl 2>&1
GSM_NO_INTERSECT=1 python tools/scale_run.py --univ ${UNIV:-100} --reps 5 --skip-oracle-above 0 > gpurun_out/isect_lubm_off.jsonl 2>&1
for f in isect_pl isect_pl_off isect_lubm isect_lubm_off; do
  echo "== $f"; python - "$f" <<'PY'
import json, sys
for l in open(f"gpurun_out/{sys.argv[1]}.jsonl"):
    try: d = json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    if "query" in d: print(d["query"], d.get("gpu_ms"), d.get("kinds"), d.get("parity"), d.get("error", ""))
PY
done
