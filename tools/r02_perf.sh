#!/usr/bin/env bash
# Round-2 performance session: parity of the changed paths, host profile,
# batch composition probe, write bandwidth, a bench line.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_chunked.py -x -q -p no:cacheprovider \
    > gpurun_out/perf_pytest.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/perf_pytest.log
python tools/write_bw.py > gpurun_out/write_bw.json 2>&1; cat gpurun_out/write_bw.json
python tools/host_profile.py > gpurun_out/host_profile.txt 2>&1; head -3 gpurun_out/host_profile.txt
python tools/batch_probe.py > gpurun_out/batch_probe.json 2>&1; cat gpurun_out/batch_probe.json
python bench.py --no-cpu-baseline --scale-univ 0 > gpurun_out/perf_bench.json 2> gpurun_out/perf_bench.err
echo "bench rc=$?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/perf_bench.json").read().strip().splitlines()[-1])
print({k: d[k] for k in ("value", "ms_per_step", "e2e", "latency_ms")})
print(json.dumps(d.get("roofline_probe"))[:1500])
PY
# ncu --set full of the output-bound expand kernels: memberOf (long rows,
# columnar -> row_warp_cols) and power-law 100M chain2 (short rows, window
# scatter, fused row-major projection)
GSM_NO_PROJ_FUSION=1 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:k_tilescan.*ExpandP" -s 3 -c 1 -o gpurun_out/prof_memberOf_cols -f \
    python bench.py --only-probe --probe memberOf_coworkers > gpurun_out/ncu_memberOf_cols.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:k_tilescan" -s 3 -c 1 -o gpurun_out/prof_pl_chain2 -f \
    python tools/pl_time.py --triples 100000000 --only chain2 --reps 5 > gpurun_out/ncu_pl_chain2.log 2>&1
python tools/ncu_summary.py gpurun_out/r02_ncu_perf.md gpurun_out/prof_memberOf_cols.ncu-rep \
    gpurun_out/prof_pl_chain2.ncu-rep > /dev/null 2>&1; cat gpurun_out/r02_ncu_perf.md | head -60
