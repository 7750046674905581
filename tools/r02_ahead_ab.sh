#!/usr/bin/env bash
set -u
cd "$(dirname "$0")/.."
python - <<'PY'
import sys, pathlib, subprocess, os; sys.path.insert(0, ".")
import bench
bench._gen_store(pathlib.Path("/tmp"), 10, 0)
if not os.path.exists("/tmp/pl100m/meta"):
    subprocess.run(["oracle/_build/gsmgen", "powerlaw", "--triples", "100000000", "--predicates", "40",
                    "--seed", "0", "--out", "/tmp/pl100m"], check=True, stdout=subprocess.DEVNULL)
PY
PREV=$PWD/paper_1807_07691_b200/_lib/libgsmat_b200_prev.so
for lib in "$PREV" "" "$PREV" ""; do
  echo "== lib=${lib:-new}"
  GSM_LIB=$lib python tools/e2e_ab.py --reps 300 --store /tmp/lubm10
  GSM_LIB=$lib python tools/pl_time.py --store /tmp/pl100m --only chain2,chain3,mix3,triangle --reps 7
  GSM_LIB=$lib python bench.py --only-probe 2>/dev/null | tail -1 | cut -c1-400
done
python -m pytest tests/test_gpu_parity.py tests/test_gpu_tables.py tests/test_gpu_chunked.py -x -q -p no:cacheprovider > gpurun_out/ahead_pytest.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/ahead_pytest.log
