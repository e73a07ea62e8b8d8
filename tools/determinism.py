"""Run-to-run determinism probe: python tools/determinism.py FRACTAL:LEVEL [steps] [reps]

Seeds the same state `reps` times, steps it `steps` times on the packed path and
prints the state hashes (all must agree); the environment selects the variant."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2110_12952_b200 import Backend, SimOptions, Simulation, conway_rule  # noqa: E402
from tools.quick_bench import DESCS  # noqa: E402


def main():
    f, level = sys.argv[1].split(":")
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    hs = []
    for _ in range(reps):
        sim = Simulation(DESCS[f], int(level), Backend.GpuCompact, SimOptions(kernel="packed", memory_cap=1 << 42))
        sim.seed_random(42, 0.5)
        h = []
        for s in range(steps):
            sim.step(conway_rule(), 1)
            h.append(sim.state_hash())
        hs.append(h)
        prog = sim.packed_program()
        sim.close()
    first = next((s for s in range(steps) if len({h[s] for h in hs}) > 1), None)
    env = {k: v for k, v in os.environ.items() if k.startswith("NBBGPU_")}
    print(f"{sys.argv[1]} {env} prog={prog} final={[f'{h[-1]:016x}'[:8] for h in hs]} first_divergence={first}", flush=True)


if __name__ == "__main__":
    main()
