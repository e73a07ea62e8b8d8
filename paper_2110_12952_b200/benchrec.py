"""The reference's benchmark harness (proj/include/nbb/bench.hpp, proj/src/bench.cpp)
on the GPU backends: BenchConfig / BenchRecord / bench_run / write_csv / read_csv
with the same CSV schema, so paper-style speedup tables (speedup_vs_bb) come out of
the same tooling.  Differences: the backends are gpu-bb / gpu-lambda / gpu-compact
(blocked when block_size > 0), each rep is timed on the device (CUDA events around
`iters` steps on the engine stream, Simulation.step_timed) instead of steady_clock,
and `kernel` selects the compact kernel.  Infeasible configurations (memory cap,
invalid block size, device memory) become skipped records, never errors
(bench.cpp:83-138).
"""
from __future__ import annotations

import csv
import io
import math
from dataclasses import dataclass, field
from typing import List, Optional, TextIO

from .descriptor import FractalDescriptor, cell_count, side_length
from .simulation import DEFAULT_MEMORY_CAP, SimOptions, Simulation
from .stencil import Backend, StencilRule, conway_rule

CSV_HEADER = ("fractal,level,n,backend,block_size,reps,iters,mean_ms,stddev_ms,"
              "mem_cells,speedup_vs_bb")  # kCsvHeader, bench.hpp:57-59


@dataclass
class BenchRecord:
    """bench.hpp:18-31"""
    fractal: str = ""
    level: int = 0
    n: int = 0
    backend: str = ""
    block_size: int = 0
    reps: int = 0
    iters: int = 0
    mean_ms: Optional[float] = None
    stddev_ms: Optional[float] = None
    mem_cells: int = 0
    speedup_vs_bb: Optional[float] = None
    skip_reason: str = ""


@dataclass
class BenchConfig:
    """bench.hpp:33-50 (GPU backends)."""
    desc: FractalDescriptor = None
    levels: List[int] = field(default_factory=list)
    backends: List[Backend] = field(default_factory=lambda: [Backend.GpuBoundingBox, Backend.GpuLambda,
                                                              Backend.GpuCompact])
    block_sizes: List[int] = field(default_factory=lambda: [0])
    reps: int = 5
    iters: int = 50
    rule: StencilRule = field(default_factory=conway_rule)
    seed: int = 42
    density: float = 0.5
    memory_cap: int = DEFAULT_MEMORY_CAP
    warmup: bool = True
    kernel: str = "auto"
    device: int = 0


def _stored_cells(desc: FractalDescriptor, level: int, backend: Backend, rho: int) -> int:
    """stored_cells (geometry.cpp:81-108) of the layout the backend uses."""
    if backend in (Backend.GpuBoundingBox, Backend.GpuLambda):
        return side_length(desc, level) ** 2
    if rho <= 0:
        return cell_count(desc, level)
    m, p = 0, 1
    while p < rho:
        p *= desc.growth
        m += 1
    if p != rho:
        raise ValueError(f"block size {rho} is not a power of s={desc.growth}")
    if m > level:
        raise ValueError(f"block size {rho} exceeds the level-{level} fractal")
    return desc.replica_count ** (level - m) * rho * rho


def _time_record(config: BenchConfig, backend: Backend, rec: BenchRecord) -> None:
    """time_record, bench.cpp:28-59, with device timing."""
    opts = SimOptions(block_size=rec.block_size, memory_cap=config.memory_cap, device=config.device,
                      kernel=config.kernel if backend == Backend.GpuCompact and rec.block_size == 0 else "auto")
    with Simulation(config.desc, rec.level, backend, opts) as sim:
        sim.seed_random(config.seed, config.density)
        if config.warmup:
            sim.step(config.rule, config.iters)
        per_iter = [sim.step_timed(config.rule, config.iters) / config.iters for _ in range(config.reps)]
    mean = sum(per_iter) / len(per_iter)
    var = sum((v - mean) ** 2 for v in per_iter) / (len(per_iter) - 1) if len(per_iter) > 1 else 0.0
    rec.mean_ms, rec.stddev_ms = mean, math.sqrt(var)


def bench_run(config: BenchConfig, progress: Optional[TextIO] = None) -> List[BenchRecord]:
    """bench.cpp:83-138: every (level, backend, block size), speedup against the
    gpu-bb row of the same level."""
    records: List[BenchRecord] = []
    for level in config.levels:
        start = len(records)
        for backend in config.backends:
            for rho in (config.block_sizes if backend == Backend.GpuCompact else [0]):
                rec = BenchRecord(config.desc.name, level, side_length(config.desc, level), backend.value,
                                  rho, config.reps, config.iters)
                tag = f" rho={rho}" if rho > 0 else ""
                try:
                    rec.mem_cells = _stored_cells(config.desc, level, backend, rho)
                    if rec.mem_cells > config.memory_cap:
                        raise ValueError(f"grid of {rec.mem_cells} cells exceeds the memory cap of "
                                         f"{config.memory_cap} bytes")
                    if progress:
                        print(f"bench: {rec.fractal} r={level} {rec.backend}{tag} ...", file=progress)
                    _time_record(config, backend, rec)
                except Exception as e:  # skipped, not fatal
                    rec.skip_reason = str(e)
                    if progress:
                        print(f"bench: skipped {rec.fractal} r={level} {rec.backend}{tag}: {e}", file=progress)
                records.append(rec)
        bb = [r.mean_ms for r in records[start:] if r.backend == Backend.GpuBoundingBox.value and r.mean_ms]
        if bb:
            for r in records[start:]:
                if r.mean_ms:
                    r.speedup_vs_bb = bb[-1] / r.mean_ms
    return records


def _fmt(v: Optional[float]) -> str:
    return "" if v is None else f"{v:.6f}"


def write_csv(records: List[BenchRecord], out: TextIO) -> None:
    """bench.cpp:140-153"""
    w = csv.writer(out, lineterminator="\n")
    out.write(CSV_HEADER + "\n")
    for r in records:
        w.writerow([r.fractal, r.level, r.n, r.backend, r.block_size if r.block_size > 0 else "-", r.reps,
                    r.iters, _fmt(r.mean_ms), _fmt(r.stddev_ms), r.mem_cells, _fmt(r.speedup_vs_bb)])


def read_csv(inp: TextIO) -> List[BenchRecord]:
    """Round-trip reader for the same schema (bench.cpp read_csv)."""
    rows = list(csv.reader(inp))
    if not rows or ",".join(rows[0]) != CSV_HEADER:
        raise ValueError("unexpected CSV header")
    out = []
    for f in rows[1:]:
        if not f:
            continue
        out.append(BenchRecord(f[0], int(f[1]), int(f[2]), f[3], 0 if f[4] == "-" else int(f[4]), int(f[5]),
                               int(f[6]), float(f[7]) if f[7] else None, float(f[8]) if f[8] else None,
                               int(f[9]), float(f[10]) if f[10] else None))
    return out


def to_csv_string(records: List[BenchRecord]) -> str:
    s = io.StringIO()
    write_csv(records, s)
    return s.getvalue()
