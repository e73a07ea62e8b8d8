"""Paper-style backend comparison tables on the GPU (bench.cpp's CSV schema):
python tools/bench_csv.py > profiles/r2_bench_backends.csv"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2110_12952_b200 import builtin_descriptor  # noqa: E402
from paper_2110_12952_b200.benchrec import BenchConfig, bench_run, write_csv  # noqa: E402

recs = []
T = builtin_descriptor("sierpinski-triangle")
C = builtin_descriptor("sierpinski-carpet")
recs += bench_run(BenchConfig(desc=T, levels=[10, 12, 14, 16], block_sizes=[0, 4, 16], reps=3, iters=20,
                              memory_cap=1 << 36), sys.stderr)
recs += bench_run(BenchConfig(desc=C, levels=[5, 7, 9], block_sizes=[0, 3, 9], reps=3, iters=20,
                              memory_cap=1 << 36), sys.stderr)
write_csv(recs, sys.stdout)
