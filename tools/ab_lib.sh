# A/B of built libraries: bash tools/ab_lib.sh [lib.so ...] (default: ab_prev.so vs the current build)
cd "$(dirname "$0")/.."
LIBS=${*:-"$PWD/paper_2110_12952_b200/ab_prev.so current"}
CASES=${AB_CASES:-"T:20:packed H:11:packed H:10:packed C:10:packed C:11:packed C:9:packed K:12:packed Y:9:packed"}
for rep in 1 2; do
  for lib in $LIBS; do
    [ "$lib" = current ] && lib=""
    echo "== lib=${lib:-current}"
    NBBGPU_LIB=$lib QB_STEPS=50 QB_PROF=1 timeout 600 python tools/quick_bench.py $CASES 2>&1 | grep -v Warn
  done
done
