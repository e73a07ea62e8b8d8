#!/usr/bin/env python3
"""Generates tests/golden/*.json from the UNMODIFIED reference library.

Producer: oracle/_ref/libnbbref.so, compiled by oracle/Makefile straight from
/root/reference/proj/src (run only in the build container, where the reference
exists).  Every value comes from nbb::Simulation's public API
(seed_random / step / state_hash / front().data(), proj/include/nbb/stencil.hpp).

Fingerprints:
  state_hash -- Simulation::state_hash() (proj/src/stencil.cpp:196-234)
  fnv        -- FNV-1a-64 over front().data() (k^r bytes cy*w+cx, or n*n for bb)

Usage: python tests/golden/make_golden.py [--big]
"""
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_2110_12952_b200.descriptor import builtin_descriptor, load_descriptor  # noqa: E402

WORKERS = os.cpu_count() or 1


def desc_of(name):
    if name.startswith("@"):
        return load_descriptor("@" + os.path.join(ROOT, name[1:]))
    if name == "solid":
        from paper_2110_12952_b200.descriptor import FractalDescriptor
        return FractalDescriptor("solid", 4, 2, [(0, 0), (1, 0), (0, 1), (1, 1)])
    return builtin_descriptor(name)


def trace(name, level, steps, backend="compact", seed=42, density=0.5, birth=0x8, survive=0xC,
          moore=True, every=1, dump_steps=(), checkpoints=None):
    d = desc_of(name)
    sim = oracle.RefSim(d.replicas, d.k, d.s, level, backend=backend, workers=WORKERS)
    sim.seed_random(seed, density)
    rec = {"fractal": name, "k": d.k, "s": d.s, "replicas": d.replicas, "level": level,
           "backend": backend, "seed": seed, "density": density, "birth": birth,
           "survive": survive, "moore": moore, "steps": {}, "dumps": {}}
    want = set(checkpoints) if checkpoints is not None else None

    def record(t):
        if (want is None and t % every == 0) or (want is not None and t in want):
            buf = sim.front()
            rec["steps"][str(t)] = {"state_hash": f"{sim.state_hash():016x}",
                                    "fnv": f"{oracle.fnv1a64(buf):016x}",
                                    "alive": int(buf.sum(dtype=np.int64))}
        if t in dump_steps:
            rec["dumps"][str(t)] = sim.front().tobytes().hex()

    record(0)
    for t in range(1, steps + 1):
        sim.step(birth, survive, moore)
        record(t)
    return rec


def splitmix_stream(seed):
    st = seed
    while True:
        yield oracle.lib().nbbo_splitmix64(st & 0xFFFFFFFFFFFFFFFF)
        st += 1


def randomized_trials(seed, n, fractals, steps, density_rand):
    """Mirrors acceptance.cpp:202-219 (SplitMix(424242), T r=4, 8 steps, density
    0.1+0.8u) and test_stencil.cpp:155-182 (SplitMix(2024), alternating T r=4 /
    carpet r=2, density 0.5): rule/seed drawn in the reference's order."""
    g = splitmix_stream(seed)
    out = []
    for trial in range(n):
        name, level = fractals(trial)
        birth = next(g) & 0x1FF
        survive = next(g) & 0x1FF
        moore = bool(next(g) & 1)
        s = next(g)
        density = 0.5
        if density_rand:
            density = 0.1 + 0.8 * ((next(g) >> 11) * (1.0 / 9007199254740992.0))
        rec = trace(name, level, steps, seed=s, density=density, birth=birth, survive=survive,
                    moore=moore)
        bb = trace(name, level, steps, backend="bb", seed=s, density=density, birth=birth,
                   survive=survive, moore=moore)
        for t in rec["steps"]:
            assert rec["steps"][t]["state_hash"] == bb["steps"][t]["state_hash"]
            rec["steps"][t]["bb_fnv"] = bb["steps"][t]["fnv"]
        out.append(rec)
    return out


def main():
    big = "--big" in sys.argv
    t0 = time.time()
    out = {"producer": "oracle/_ref/libnbbref.so (unmodified reference sources)",
           "traces": [], "random_c5": [], "random_xbackend": []}
    # small configs: every step, compact + bb
    for name, level, steps, dumps in [("sierpinski-triangle", 6, 100, (0, 1, 2, 3, 10)),
                                      ("sierpinski-triangle", 10, 100, ()),
                                      ("sierpinski-carpet", 5, 100, ()),
                                      ("vicsek", 6, 100, ()),
                                      ("@descriptors/h-fractal.desc", 6, 100, ()),
                                      ("@descriptors/candy.desc", 5, 100, ()),
                                      ("solid", 5, 20, ()),
                                      ("sierpinski-triangle", 1, 5, (0, 1)),
                                      ("sierpinski-triangle", 0, 3, (0, 1))]:
        rec = trace(name, level, steps, dump_steps=dumps)
        bbrec = trace(name, level, steps, backend="bb",
                      dump_steps=dumps if level <= 6 else ())
        for t in rec["steps"]:
            assert rec["steps"][t]["state_hash"] == bbrec["steps"][t]["state_hash"], (name, t)
            rec["steps"][t]["bb_fnv"] = bbrec["steps"][t]["fnv"]
        rec["bb_dumps"] = bbrec["dumps"]
        out["traces"].append(rec)
        print(f"{name} r={level}: {time.time() - t0:.1f}s", flush=True)

    # von Neumann + a B0 rule on the triangle (holes must stay dead)
    for birth, survive, moore in [(0x1FF, 0x1FF, True), (0x6, 0x9, False), (0x1, 0x0, True)]:
        rec = trace("sierpinski-triangle", 7, 12, birth=birth, survive=survive, moore=moore)
        bbrec = trace("sierpinski-triangle", 7, 12, backend="bb", birth=birth, survive=survive,
                      moore=moore)
        for t in rec["steps"]:
            assert rec["steps"][t]["state_hash"] == bbrec["steps"][t]["state_hash"]
            rec["steps"][t]["bb_fnv"] = bbrec["steps"][t]["fnv"]
        out["traces"].append(rec)

    out["random_c5"] = randomized_trials(424242, 50, lambda t: ("sierpinski-triangle", 4), 8, True)
    out["random_xbackend"] = randomized_trials(
        2024, 15, lambda t: ("sierpinski-triangle", 4) if t % 2 == 0 else ("sierpinski-carpet", 2),
        6, False)
    print(f"random trials: {time.time() - t0:.1f}s", flush=True)

    # medium levels: checkpoints only
    out["traces"].append(trace("sierpinski-triangle", 13, 4, checkpoints=(0, 1, 4)))
    out["traces"].append(trace("sierpinski-triangle", 14, 3, checkpoints=(0, 1, 3)))
    out["traces"].append(trace("sierpinski-carpet", 7, 10, checkpoints=(0, 1, 2, 10)))
    if big:
        out["traces"].append(trace("sierpinski-triangle", 16, 10, checkpoints=(0, 1, 2, 3, 10)))
        out["traces"].append(trace("sierpinski-carpet", 9, 2, checkpoints=(0, 1, 2)))
    print(f"done: {time.time() - t0:.1f}s", flush=True)
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(out, fh, indent=0, sort_keys=True)


if __name__ == "__main__":
    main()
