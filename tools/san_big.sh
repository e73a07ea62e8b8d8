cd "$(dirname "$0")/.."
OUT=gpurun_out/sanitize; mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
for c in jit_k11 carpet_c10; do
  for tool in initcheck memcheck racecheck; do
    extra=""; [ $tool = racecheck ] && extra="--racecheck-report hazard"
    timeout 900 $CS --tool $tool $extra --print-limit 30 python tools/sanitize_run.py $c > $OUT/${tool}_$c.log 2>&1
    echo "$tool $c rc=$? | $(grep -E "^$c: " $OUT/${tool}_$c.log | tail -1) | $(grep -E "ERROR SUMMARY|RACECHECK SUMMARY" $OUT/${tool}_$c.log | tail -1)"
  done
done
