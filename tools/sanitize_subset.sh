#!/bin/bash
# compute-sanitizer over a subset of tools/sanitize_run.py cases:
#   SAN_CASES="a b" tools/sanitize_subset.sh [tool ...]
set -u
cd "$(dirname "$0")/.."
OUT=gpurun_out/sanitize; mkdir -p $OUT
TOOLS=${*:-memcheck synccheck racecheck}
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in $TOOLS; do
  for c in $SAN_CASES; do
    extra=""
    [ $tool = racecheck ] && extra="--racecheck-report all"
    timeout 900 $CS --tool $tool $extra --print-limit 20 python tools/sanitize_run.py $c > $OUT/${tool}_$c.log 2>&1
    rc=$?
    summ=$(grep -E "ERROR SUMMARY|RACECHECK SUMMARY" $OUT/${tool}_$c.log | tail -1)
    res=$(grep -E "^$c: " $OUT/${tool}_$c.log | tail -1)
    echo "$tool $c rc=$rc | $res | $summ" | tee -a $OUT/summary.txt
  done
done
