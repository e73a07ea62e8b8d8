for lib in "" "$PWD/abprev.so"; do
  echo "== lib=${lib:-current}"
  for g in 0 1; do NBBGPU_LIB=$lib NBBGPU_GRAPHS=$g QB_STEPS=50 timeout 300 python tools/quick_bench.py T:20:packed T:18:packed T:16:packed 2>&1 | tail -3 | sed "s/^/graphs=$g /"; done
done
