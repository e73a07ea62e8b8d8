"""Where two runs of the same seeded state part ways: python tools/divergence.py [FRACTAL:LEVEL] [steps]
(several FRACTAL:LEVEL:STEPS arguments sweep configurations in one process)

With DIV_PREAMBLE=1 first replays tools/quick_bench.py's preamble (other states created, stepped and freed in
the same process), then steps three handles of FRACTAL:LEVEL in lockstep -- A through
step_profiled, B through step, R on the table-driven program (NBBGPU_JIT=0) -- and
at the first hash mismatch reports the differing compact cells (tile, group, local
position)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2110_12952_b200 import Backend, SimOptions, Simulation, conway_rule  # noqa: E402
from tools.quick_bench import DESCS  # noqa: E402


def make(f, level, env=None):
    saved = {k: os.environ.get(k) for k in (env or {})}
    os.environ.update(env or {})
    try:
        s = Simulation(DESCS[f], level, Backend.GpuCompact, SimOptions(kernel="packed", memory_cap=1 << 42))
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    return s


def main():
    if len(sys.argv) > 1 and sys.argv[1].count(":") == 2:  # sweep
        for case in sys.argv[1:]:
            f, level, steps = case.split(":")
            lockstep(f, int(level), int(steps))
        return
    f, level = (sys.argv[1] if len(sys.argv) > 1 else "K:12").split(":")
    lockstep(f, int(level), int(sys.argv[2]) if len(sys.argv) > 2 else 60)


def lockstep(f, level, steps):
    rule = conway_rule()
    if os.environ.get("DIV_PREAMBLE"):
        for case in ("T:20", "H:11", "H:10", "C:10", "C:11", "C:9"):
            pf, pl = case.split(":")
            s = make(pf, int(pl))
            s.seed_random(42, 0.5)
            s.step(rule, 3)
            s.step_timed(rule, 50)
            s.step_profiled(rule, 50)
            s.close()
    A, B, R = make(f, level), make(f, level), make(f, level, {"NBBGPU_JIT": "0", "NBBGPU_GENERIC": "1"})
    print(f"{f}:{level} programs", A.packed_program(), B.packed_program(), R.packed_program(), flush=True)
    for s in (A, B, R):
        s.seed_random(42, 0.5)
    d = DESCS[f]
    W = d.k ** ((level + 1) // 2)
    for i in range(steps):
        A.step_profiled(rule, 1)
        B.step(rule, 1)
        R.step(rule, 1)
        ha, hb, hr = A.state_hash(), B.state_hash(), R.state_hash()
        if ha == hb == hr:
            continue
        print(f"step {i + 1}: A {ha:016x} B {hb:016x} R {hr:016x}", flush=True)
        ref = R.front().data
        for name, s, h in (("A", A, ha), ("B", B, hb)):
            if h == hr:
                continue
            diff = np.nonzero(s.front().data != ref)[0]
            x, y = diff % W, diff // W
            wq = 36 if f == "K" else None
            print(f"  {name}: {diff.size} cells differ; first {diff[:10].tolist()}", flush=True)
            if wq:
                t = (y // wq) * (W // wq) + x // wq
                print(f"  tiles {np.unique(t)[:20].tolist()} groups {np.unique(t // 32)[:20].tolist()} "
                      f"local {list(zip((x % wq)[:10].tolist(), (y % wq)[:10].tolist()))}", flush=True)
        break
    else:
        print(f"{f}:{level} no divergence in {steps} steps ({ha:016x})", flush=True)
    for s in (A, B, R):
        s.close()


if __name__ == "__main__":
    main()
