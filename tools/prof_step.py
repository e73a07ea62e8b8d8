#!/usr/bin/env python3
"""Profiling driver: seed + a few steps of one configuration (used under ncu)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2110_12952_b200 import (Backend, SimOptions, Simulation, StencilRule,  # noqa: E402
                                   builtin_descriptor, load_descriptor)

ap = argparse.ArgumentParser()
ap.add_argument("--fractal", default="sierpinski-triangle")
ap.add_argument("--level", type=int, default=20)
ap.add_argument("--steps", type=int, default=4)
ap.add_argument("--backend", default="gpu-compact")
ap.add_argument("--kernel", default="auto")
ap.add_argument("--rule", default="B3/S23")
a = ap.parse_args()
d = load_descriptor(a.fractal) if a.fractal.startswith("@") else builtin_descriptor(a.fractal)
b = Backend.GpuCompact if a.backend == "gpu-compact" else Backend.GpuBoundingBox
sim = Simulation(d, a.level, b, SimOptions(memory_cap=1 << 42, kernel=a.kernel))
sim.seed_random(42, 0.5)
ms = sim.step_timed(StencilRule.parse(a.rule), a.steps)
print(f"{a.fractal} r={a.level} {a.backend} {sim.active_kernel()}: {ms / a.steps:.3f} ms/step, "
      f"{d.k ** a.level * a.steps / (ms / 1e3):.3e} cell-updates/s, hash={sim.state_hash():016x}")
