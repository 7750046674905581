#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
make -s -C oracle
python tools/scale_run.py --kind powerlaw --triples 1000000000 --store /tmp/pl1b \
    --only star4,chain2,chain3,triangle,self_chain --summary star4 --reps 3 \
    --skip-oracle-above 0 > gpurun_out/r02_pl1b.jsonl 2> gpurun_out/r02_pl1b.err
echo "rc=$?"; cut -c1-700 gpurun_out/r02_pl1b.jsonl; tail -3 gpurun_out/r02_pl1b.err
