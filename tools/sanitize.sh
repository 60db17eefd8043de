#!/bin/bash
# compute-sanitizer over every kernel family of libjoinqr.so at C1/C2-shaped sizes
# (tools/sanitize_run.py).  Logs -> gpurun_out/sanitize_<tool>.log; summary at the end.
# Usage (GPU box): bash tools/sanitize.sh [tools...]
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
TOOLS=${*:-memcheck racecheck synccheck initcheck}
for t in $TOOLS; do
  extra=""
  [ "$t" = memcheck ] && extra="--leak-check full"
  [ "$t" = racecheck ] && extra="--racecheck-report all"
  echo "== $t" | tee gpurun_out/sanitize_$t.log
  timeout 1500 $CS --tool $t $extra --target-processes all --print-limit 50 \
      python tools/sanitize_run.py all >> gpurun_out/sanitize_$t.log 2>&1
  echo "exit $?" >> gpurun_out/sanitize_$t.log
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|LEAK SUMMARY|sanitize_run done|^exit" gpurun_out/sanitize_$t.log
done
