#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
python tools/scale_run.py --kind lubm --univ 1000 --store /tmp/lubm1000 --skip-oracle-above 0 --reps 5 \
   --only q02,q08,q09,c1_advisor_course_triangle,c2_dept_univ_alumni_triangle,c3_coauthor_advisor,c4_snowflake,c7_ta_of_advisor_course,c8_research_chain \
   2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if 'query' in d: print(d['query'], d.get('gpu_ms'), d.get('kinds'))
"
python - <<'PY'
import subprocess, os
if not os.path.exists("/tmp/pl100m/meta"):
    subprocess.run(["oracle/_build/gsmgen", "powerlaw", "--triples", "100000000", "--predicates", "40",
                    "--seed", "0", "--out", "/tmp/pl100m"], check=True, stdout=subprocess.DEVNULL)
PY
python tools/pl_time.py --store /tmp/pl100m --only triangle,mix3 --reps 7
