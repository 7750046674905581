#!/usr/bin/env bash
# Round-2 profiling pass: launch list (+ DRAM bytes per launch) of a bench
# run, ncu --set full of q09's fused groups and a filter.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/r02_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-probe --scale-univ 0 --scale-watdiv 0 > gpurun_out/ncu_launch.log 2>&1
python tools/traffic_from_csv.py gpurun_out/r02_launches.csv gpurun_out/ncu_traffic.json
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:k_group -s 6 -c 2 \
    -o gpurun_out/prof_q09_group -f python tools/query_ncu.py q09 --reps 6 > gpurun_out/ncu_q09.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:FilterP -s 3 -c 1 \
    -o gpurun_out/prof_q01_filter -f python tools/query_ncu.py q01 --reps 6 > gpurun_out/ncu_q01.log 2>&1
python tools/ncu_summary.py gpurun_out/r02_ncu_full.md gpurun_out/r02_launches.csv \
    gpurun_out/prof_q09_group.ncu-rep gpurun_out/prof_q01_filter.ncu-rep
head -30 gpurun_out/r02_ncu_full.md
