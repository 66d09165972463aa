#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over every
# kernel family at small shapes (profiles/scripts/sanitize_cases.py).
# Usage: bash profiles/scripts/sanitize.sh <outdir>
set -u
OUT=${1:-gpurun_out/sanitize}
mkdir -p "$OUT"
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check full"
  [ "$tool" = racecheck ] && extra="--racecheck-report all"
  timeout 1500 $CS --tool $tool $extra --target-processes all --print-limit 200 \
     --error-exitcode 99 python profiles/scripts/sanitize_cases.py > "$OUT/$tool.log" 2>&1
  echo "$tool rc=$?" | tee -a "$OUT/summary.txt"
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|LEAK SUMMARY" "$OUT/$tool.log" | tail -3 | tee -a "$OUT/summary.txt"
done
