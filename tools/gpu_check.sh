#!/usr/bin/env bash
# One GPU session: the -m gpu suite, sanitizers, smoke, bench (both arms).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest_rc=$?"; tail -4 gpurun_out/pytest_gpu.log
[ "${SANITIZE:-1}" = 1 ] && bash tools/sanitize.sh
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
if [ "${BENCH:-1}" = 1 ]; then
  python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench_rc=$?"
  tail -c 3000 gpurun_out/bench.json
  python bench.py --impl reference --steps ${REF_STEPS:-5} --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
  echo "ref_rc=$?"; tail -c 1500 gpurun_out/bench_ref.json
fi
