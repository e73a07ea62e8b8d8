"""Quick device timing of the step kernels: python tools/quick_bench.py [fractal:level:kernel ...]

Prints ms/step (CUDA events around nsteps launches on the engine stream), cell-updates/s
and the final state hash for each case (default: T r=20 packed and tiled).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2110_12952_b200 import (Backend, SimOptions, Simulation, builtin_descriptor,  # noqa: E402
                                   conway_rule)
from paper_2110_12952_b200.descriptor import FractalDescriptor  # noqa: E402

DESCS = {
    "T": builtin_descriptor("sierpinski-triangle"),
    "C": builtin_descriptor("sierpinski-carpet"),
    "V": builtin_descriptor("vicsek"),
    "H": FractalDescriptor("h-fractal", 7, 3, [(0, 0), (2, 0), (0, 1), (1, 1), (2, 1), (0, 2), (2, 2)]),
    "Y": FractalDescriptor("candy", 12, 4, [(1, 0), (2, 0), (0, 1), (1, 1), (2, 1), (3, 1), (0, 2),
                                            (1, 2), (2, 2), (3, 2), (1, 3), (2, 3)]),
    # a descriptor with no compile-time wiring (generic transition-table program)
    "K": FractalDescriptor("k6s3", 6, 3, [(0, 0), (1, 0), (2, 0), (0, 1), (1, 2), (2, 2)]),
}


def main(cases):
    rule = conway_rule()
    for case in cases:
        f, level, kernel = case.split(":")
        level = int(level)
        d = DESCS[f]
        if kernel == "bb":  # the bounding-box baseline
            sim = Simulation(d, level, Backend.GpuBoundingBox, SimOptions(memory_cap=1 << 42))
        else:
            sim = Simulation(d, level, Backend.GpuCompact, SimOptions(kernel=kernel, memory_cap=1 << 42))
        sim.seed_random(42, 0.5)
        sim.step(rule, 3)
        steps = int(os.environ.get("QB_STEPS", "20"))
        ms = sim.step_timed(rule, steps) / steps
        cells = d.k ** level
        extra = ""
        if kernel == "bb":
            extra = f" | BB dense model {2 * d.s ** (2 * level) / (ms / 1e3) / 1e9:.0f} GB/s"
        if os.environ.get("QB_PROF"):
            tot, main, n = sim.step_profiled(rule, steps)
            extra = f" | step kernel {main / steps * 1e3:.1f} us of {tot / steps * 1e3:.1f} us, {n / steps:.0f} launches/step"
        print(f"{case:14s} {sim.active_kernel() if kernel != 'bb' else 'bb'} {ms:9.4f} ms/step {cells * 1e3 / ms:10.3e} cell-updates/s "
              f"hash={sim.state_hash():016x} held={sim.peak_bytes() / 1e9:.3f} GB{extra}", flush=True)
        sim.close()


if __name__ == "__main__":
    main(sys.argv[1:] or ["T:20:packed", "T:20:tiled"])
