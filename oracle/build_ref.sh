#!/usr/bin/env bash
# Installs the UNMODIFIED reference package (pure Python, stdlib only) from
# /root/reference into oracle/_ref so it can act as the "reference" CPU arm
# (bench.py --impl reference) and as the parity checker on the GPU box, where
# /root/reference does not exist.  oracle/_ref is git-ignored (never committed)
# but travels with the gpurun snapshot.  No reference source is copied into
# the repository itself.
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
src="${1:-/root/reference/pkg}"
if [ ! -d "$src" ]; then
  echo "build_ref.sh: reference not present at $src; keeping existing oracle/_ref" >&2
  exit 0
fi
tmp="$(mktemp -d)"
trap 'rm -rf "$tmp"' EXIT
cp -r "$src" "$tmp/pkg"          # the reference tree is read-only; build from a copy
rm -rf "$here/_ref"
python -m pip install --quiet --no-index --no-build-isolation --no-deps \
  --target "$here/_ref" "$tmp/pkg"
# the reference's own test modules (run against the drop-in by
# tests/test_reference_suite.py through the INTEGRATION.md §2 patch)
cp -r "$tmp/pkg/tests" "$here/_ref/gsmat_tests"
echo "installed reference gsmat (+ its tests) into $here/_ref"
