#!/usr/bin/env bash
# configs[4]: power-law 1B triples on one B200, current kernels, with the C
# oracle on every query whose steps fit host RAM (exact row compare up to
# 100M rows, fingerprints above), star4 through execute_summary.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
make -s -C oracle
timeout 2700 python tools/scale_run.py --kind powerlaw --triples 1000000000 \
    --summary star4 --reps 3 --skip-oracle-above 600000000 --exact-rows 100000000 \
    > gpurun_out/r02_pl1b_parity.jsonl 2> gpurun_out/r02_pl1b_parity.err
echo "rc=$?"; cut -c1-400 gpurun_out/r02_pl1b_parity.jsonl; tail -3 gpurun_out/r02_pl1b_parity.err
