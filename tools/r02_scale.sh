#!/usr/bin/env bash
# Round-2 scale runs (GPU box): T4 skew store, WatDiv C2 and power-law-1B
# star4 through left-row chunking / execute_summary.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
make -s -C oracle
python tools/scale_run.py --kind powerlaw --triples 100000000 --node-skew 0.9 --qdir powerlaw_skew \
    --summary self_chain_hubs --reps 5 > gpurun_out/r02_scale_skew.jsonl 2> gpurun_out/r02_scale_skew.err
echo "skew rc=$?"; tail -c 1500 gpurun_out/r02_scale_skew.jsonl
python tools/scale_run.py --kind watdiv --scale 1000 --only C1,C2 --summary C2 --reps 3 \
    > gpurun_out/r02_scale_watdiv_c2.jsonl 2> gpurun_out/r02_scale_watdiv_c2.err
echo "watdiv rc=$?"; tail -c 1500 gpurun_out/r02_scale_watdiv_c2.jsonl
if [ "${PL1B:-1}" = 1 ]; then
  python tools/scale_run.py --kind powerlaw --triples 1000000000 --only star4,chain2,triangle \
      --summary star4 --reps 3 > gpurun_out/r02_scale_pl1b.jsonl 2> gpurun_out/r02_scale_pl1b.err
  echo "pl1b rc=$?"; tail -c 2000 gpurun_out/r02_scale_pl1b.jsonl
fi
