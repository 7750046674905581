#!/usr/bin/env bash
# A/B of the pipelined candidate loads in k_group's block-cooperative count
# against the previous build: LUBM-10 (l2_probe) and LUBM-1000 (bench scale_lubm).
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B=paper_1807_07691_b200/_lib/libgsmat_b200_base.so
N=paper_1807_07691_b200/_lib/libgsmat_b200.so
for lib in $B $N $B $N; do
  GSM_LIB=$PWD/$lib timeout 300 python tools/l2_probe.py --label "$(basename $lib)" >> gpurun_out/pipe_ab.jsonl 2>> gpurun_out/pipe_ab.err
done
python - <<'PY'
import json
for l in open("gpurun_out/pipe_ab.jsonl"):
    r = json.loads(l); c = r["cold"]
    print(f'{r["label"]:28s} batch {c["batch"]} q02 {c["q02"]} q08 {c["q08"]} q09 {c["q09"]} sum {round(sum(v for k, v in c.items() if k != "batch"), 4)}')
PY
for lib in $B $N; do
  GSM_LIB=$PWD/$lib python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-probe --scale-watdiv 0 > gpurun_out/pipe_bench_$(basename $lib).json 2>/dev/null
  python - "$lib" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/pipe_bench_{sys.argv[1].split('/')[-1]}.json").read().strip().splitlines()[-1])
q = d["scale_lubm"]["queries"]
print(sys.argv[1].split('/')[-1], "parity", d["scale_lubm"]["parity"]["ok"], "total", d["scale_lubm"]["total"]["ms"],
      {k: q[k]["ms"] for k in ("q02", "q09", "c1_advisor_course_triangle", "c2_dept_univ_alumni_triangle", "c4_snowflake", "c6_same_degree_univ", "c8_research_chain")})
PY
done
python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "variants or golden or lubm" 2>&1 | tail -1
