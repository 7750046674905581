#!/usr/bin/env bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over
# tools/sanitize_cases.py.  Logs to gpurun_out/sanitize_<tool>.log
set -uo pipefail
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CS=${CS:-/usr/local/cuda/bin/compute-sanitizer}
rc_all=0
for tool in memcheck racecheck synccheck initcheck; do
  n=30
  [ "$tool" = racecheck ] && n=12
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check full"
  timeout 1500 "$CS" --tool "$tool" $extra --error-exitcode 99 --print-limit 50 \
      python tools/sanitize_cases.py "$n" > "gpurun_out/sanitize_${tool}.log" 2>&1
  rc=$?
  # every block walking many tiles (count-ahead schedule, cross-block look-back)
  GSM_GRID_MAX=3 timeout 1500 "$CS" --tool "$tool" $extra --error-exitcode 99 --print-limit 50 \
      python tools/sanitize_cases.py 4 >> "gpurun_out/sanitize_${tool}.log" 2>&1
  rc2=$?
  [ $rc -eq 0 ] && rc=$rc2
  echo "$tool rc=$rc $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize cases' gpurun_out/sanitize_${tool}.log | tr '\n' ' ')"
  [ $rc -ne 0 ] && rc_all=$rc
done
exit $rc_all
