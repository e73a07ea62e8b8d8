"""Per-rank step cost of a partitioned T r=20 run, measured on one GPU: a handle
partitioned as rank 0 of N (no transport attached) steps only its 1/N of the groups
(halo-words + step kernel).  This is the compute part of one step at N GPUs; the
peer push and counter wait come on top (projection, not a multi-GPU measurement)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2110_12952_b200 import (Backend, SimOptions, Simulation, builtin_descriptor,  # noqa: E402
                                   conway_rule, _abi)

T = builtin_descriptor("sierpinski-triangle")
level = int(sys.argv[1]) if len(sys.argv) > 1 else 20
base = None
for n in (1, 2, 4, 8):
    sim = Simulation(T, level, Backend.GpuCompact, SimOptions(memory_cap=1 << 42))
    sim.seed_random(42, 0.5)
    if n > 1:
        _abi.check(_abi.lib().nbbgpu_partition(sim.handle(), 0, n))
    sim.step(conway_rule(), 3)
    ms = sim.step_timed(conway_rule(), 40) / 40
    base = base or ms
    print(f"r={level} ranks={n}: {ms * 1e3:.1f} us/step per rank (compute), ideal-scaling {base / ms:.2f}x")
    sim.close()
