"""CPU: the GPU bench harness keeps the reference's CSV schema (bench.cpp
write_csv / read_csv round trip) and records infeasible configurations as skipped
(bench.cpp:83-138, test_bench.cpp:74-106) without touching a GPU."""
import io

from paper_2110_12952_b200 import builtin_descriptor
from paper_2110_12952_b200.benchrec import (CSV_HEADER, BenchConfig, BenchRecord, bench_run, read_csv,
                                            write_csv)
from paper_2110_12952_b200.stencil import Backend


def test_csv_round_trip():
    recs = [BenchRecord("sierpinski-triangle", 6, 64, "gpu-bb", 0, 3, 10, 1.5, 0.1, 4096, 1.0),
            BenchRecord("a,b \"q\"", 6, 64, "gpu-compact", 16, 3, 10, 0.5, None, 729, 3.0),
            BenchRecord("x", 7, 128, "gpu-compact", 4, 3, 10, None, None, 0, None, "skipped")]
    s = io.StringIO()
    write_csv(recs, s)
    assert s.getvalue().splitlines()[0] == CSV_HEADER
    back = read_csv(io.StringIO(s.getvalue()))
    for a, b in zip(recs, back):
        assert (a.fractal, a.level, a.n, a.backend, a.block_size, a.mem_cells) == \
               (b.fractal, b.level, b.n, b.backend, b.block_size, b.mem_cells)
        assert (a.mean_ms is None) == (b.mean_ms is None)


def test_invalid_block_sizes_are_skipped_not_fatal():
    # test_bench.cpp:74-106: {0, 2, 3, 16} at r=2 -> 3 is not a power of s, 16 > n;
    # a tiny memory cap skips every configuration before any GPU work
    cfg = BenchConfig(desc=builtin_descriptor("sierpinski-triangle"), levels=[2],
                      backends=[Backend.GpuCompact], block_sizes=[0, 2, 3, 16], memory_cap=4)
    recs = bench_run(cfg)
    assert [r.block_size for r in recs] == [0, 2, 3, 16]
    assert all(r.skip_reason and r.mean_ms is None for r in recs)
    assert "not a power of s" in recs[2].skip_reason
    assert "exceeds the level" in recs[3].skip_reason
    assert "memory cap" in recs[0].skip_reason
