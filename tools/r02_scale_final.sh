#!/usr/bin/env bash
# Closing scale runs on the final kernels: power-law 1B (configs[4] model),
# the T4 skew store, WatDiv-1000 (configs[3]) incl. C2 through chunks.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
make -s -C oracle
python tools/scale_run.py --kind watdiv --scale 1000 --summary C2 --reps 3 \
    > gpurun_out/r02f_watdiv.jsonl 2> gpurun_out/r02f_watdiv.err
echo "watdiv rc=$?"; tail -1 gpurun_out/r02f_watdiv.jsonl
python tools/scale_run.py --kind powerlaw --triples 100000000 --node-skew 0.9 --qdir powerlaw_skew \
    --summary self_chain_hubs --reps 5 > gpurun_out/r02f_skew.jsonl 2> gpurun_out/r02f_skew.err
echo "skew rc=$?"; tail -1 gpurun_out/r02f_skew.jsonl
python tools/scale_run.py --kind powerlaw --triples 1000000000 --summary star4 --reps 3 \
    --skip-oracle-above 0 > gpurun_out/r02f_pl1b.jsonl 2> gpurun_out/r02f_pl1b.err
echo "pl1b rc=$?"; cut -c1-300 gpurun_out/r02f_pl1b.jsonl
