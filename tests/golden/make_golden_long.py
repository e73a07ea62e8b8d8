#!/usr/bin/env python3
"""Long-run / large-level state hashes from the UNMODIFIED reference (oracle/_ref).

Writes tests/golden/golden_long.json.  Slow (tens of minutes on 8 cores): the
reference's neighbour-table backend (SimOptions.neighbor_table, same results,
stencil.cpp:340-352) is used for the long T r=16 run; r >= 18 levels are seeded
with the shim's parallel seeding (identical values to seed_random, which is
single-threaded in the reference) and stepped with the plain compact backend.
These values reproduce SURVEY.md 8(c)'s table, which was produced the same way.
"""
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2110_12952_b200.descriptor import builtin_descriptor, load_descriptor  # noqa: E402

W = os.cpu_count() or 1


def run(desc, level, checkpoints, table=False, parallel_seed=False):
    sim = oracle.RefSim(desc.replicas, desc.k, desc.s, level, backend="compact", workers=W,
                        neighbor_table=table)
    if parallel_seed:
        sim.parallel_seed(42, 0.5, W)
    else:
        sim.seed_random(42, 0.5)
    out = {}
    t = 0
    for cp in sorted(checkpoints):
        if cp > t:
            sim.step(0x8, 0xC, True, cp - t)
            t = cp
        out[str(cp)] = f"{sim.state_hash():016x}"
        print(desc.name, level, cp, out[str(cp)], flush=True)
    return {"fractal": desc.name, "k": desc.k, "s": desc.s, "replicas": desc.replicas,
            "level": level, "seed": 42, "density": 0.5, "birth": 8, "survive": 12, "moore": True,
            "state_hash": out}


def main():
    which = sys.argv[1:] or ["t16", "c9", "t18", "h10", "y8", "h11", "y9", "t20"]
    path = os.path.join(HERE, "golden_long.json")
    data = json.load(open(path)) if os.path.exists(path) else {}
    T = builtin_descriptor("sierpinski-triangle")
    Cd = builtin_descriptor("sierpinski-carpet")
    H = load_descriptor("@" + os.path.join(ROOT, "descriptors/h-fractal.desc"))
    Y = load_descriptor("@" + os.path.join(ROOT, "descriptors/candy.desc"))
    jobs = {
        "t16": lambda: run(T, 16, [0, 1, 3, 10, 100, 500, 1000], table=True),
        "c9": lambda: run(Cd, 9, [0, 1, 2, 10, 100, 500], table=True),
        "t18": lambda: run(T, 18, [0, 1, 2, 3, 5, 10], parallel_seed=True),
        "h10": lambda: run(H, 10, [0, 1], parallel_seed=True),
        "y8": lambda: run(Y, 8, [0, 1], parallel_seed=True),
        "h11": lambda: run(H, 11, [0, 1, 2], parallel_seed=True),
        "y9": lambda: run(Y, 9, [0, 1, 2], parallel_seed=True),
        "t20": lambda: run(T, 20, [0, 1, 2, 3, 5, 10], parallel_seed=True),
    }
    for key in which:
        t0 = time.time()
        data[key] = jobs[key]()
        data[key]["seconds"] = round(time.time() - t0, 1)
        with open(path, "w") as fh:
            json.dump(data, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
