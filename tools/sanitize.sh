#!/bin/bash
# compute-sanitizer over every hot kernel family (tools/sanitize_run.py cases).
# Usage: tools/sanitize.sh [tool ...]   (default: memcheck synccheck racecheck initcheck)
# Writes gpurun_out/sanitize/<tool>_<case>.log and a summary line per run.
set -u
cd "$(dirname "$0")/.."
OUT=gpurun_out/sanitize; mkdir -p $OUT
TOOLS=${*:-memcheck synccheck racecheck initcheck}
CASES="$(python -c "import sys; sys.path.insert(0,'tools'); import sanitize_run as s; print(' '.join(s.CASES))") maps"
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in $TOOLS; do
  for c in $CASES; do
    extra=""
    [ $tool = racecheck ] && extra="--racecheck-report all"
    timeout 600 $CS --tool $tool $extra --print-limit 20 python tools/sanitize_run.py $c > $OUT/${tool}_$c.log 2>&1
    rc=$?
    summ=$(grep -E "ERROR SUMMARY|RACECHECK SUMMARY" $OUT/${tool}_$c.log | tail -1)
    res=$(grep -E "^$c: " $OUT/${tool}_$c.log | tail -1)
    echo "$tool $c rc=$rc | $res | $summ" | tee -a $OUT/summary.txt
  done
done
