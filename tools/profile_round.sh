#!/usr/bin/env bash
# Profiling pass for one round (run on the GPU box via gpurun):
#   1. launch list of one bench step (every kernel with its device time),
#   2. ncu --set full of the dominant LUBM kernels (q09's fused groups, a
#      filter, an expand),
#   3. ncu --set full of the at-scale expand probes.
# Outputs under gpurun_out/; summarise locally with tools/ncu_summary.py and
# tools/ncu_sass_top.py.
set -u
out=gpurun_out
mkdir -p $out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-probe > $out/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:k_group -s 4 -c 2 \
    -o $out/prof_q09_group python tools/query_ncu.py q09 > $out/ncu_q09.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:FilterP -s 30 -c 2 \
    -o $out/prof_filter python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-probe \
    > $out/ncu_filter.log 2>&1
# skip the first launches of each probe (the first execution may overflow the
# arena and re-run): capture a steady-state launch
for p in memberOf_coworkers takesCourse_classmates; do
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_tilescan.*ExpandP" -s 3 -c 1 \
      -o $out/prof_probe_$p python bench.py --only-probe --probe $p > $out/ncu_probe_$p.log 2>&1
done
echo done
