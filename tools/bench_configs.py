#!/usr/bin/env python3
"""All BASELINE.json configs on one GPU (secondary measurements; bench.py is the
headline).  Device-timed with CUDA events on the engine stream after warm-up;
inputs larger than L2 except where noted.  Writes one JSON object to stdout.

  configs[0] T r=10, 100 steps, compact vs BB (launch-bound, CPU-runnable)
  configs[1] T r=16, compact; paper's per-cell kernel with CUDA-core vs tensor-core
             maps; batched lambda/nu maps/s for both variants
  configs[2] carpet r=9, compact vs GPU BB
  configs[3] T r=20 (bench.py) + T r=18 compact vs vectorised BB (largest BB level)
  configs[4] H-fractal r=11 (1.98e9 cells) and Candy r=9 (5.2e9) compact: built-in
             micro-block wiring, the same wiring compiled at run time (NVRTC, the path
             every custom descriptor takes; NBBGPU_JIT_FORCE=1), the table-driven
             program (NBBGPU_GENERIC=1), and a custom descriptor K(n,6,3) at r=12
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2110_12952_b200 import (Backend, SimOptions, Simulation, builtin_descriptor,  # noqa: E402
                                   conway_rule, load_descriptor)
from paper_2110_12952_b200.descriptor import FractalDescriptor  # noqa: E402

RULE = conway_rule()


def dev_mem_used():
    free, total = torch.cuda.mem_get_info()
    return total - free


def run(desc, level, backend=Backend.GpuCompact, steps=10, warmup=3, kernel="auto", maps="digit", env=None):
    torch.cuda.synchronize()
    m0 = dev_mem_used()
    saved = {k: os.environ.get(k) for k in (env or {})}
    os.environ.update(env or {})
    try:
        sim = Simulation(desc, level, backend, SimOptions(memory_cap=1 << 42, kernel=kernel, map_variant=maps))
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    sim.seed_random(42, 0.5)
    sim.step(RULE, warmup)
    ms = sim.step_timed(RULE, steps)
    m1 = dev_mem_used()
    cells = desc.k ** level
    out = {"fractal": desc.name, "level": level, "backend": backend.value,
           "kernel": ("%s q=%d" % sim.active_kernel() + (" (%s P=%d)" % sim.packed_program()
                                                         if sim.active_kernel()[0] == "packed" else ""))
           if backend == Backend.GpuCompact else
           ("bb-rows (row-streaming, hole skipping)" if desc.s ** level >= 32 else "bb-naive"),
           "env": env or {},
           "maps": maps, "steps": steps, "ms_per_step": ms / steps,
           "cell_updates_per_s": cells * steps / (ms / 1e3), "compact_cells": cells,
           "device_bytes_held": sim.peak_bytes(), "device_mem_delta": m1 - m0,
           "state_hash": f"{sim.state_hash():016x}"}
    if backend == Backend.GpuCompact:
        out["hbm_gbs_2B_model"] = 2 * cells / (ms / steps / 1e3) / 1e9
        if sim.active_kernel()[0] == "packed":
            out["hbm_gbs_packed_model"] = 0.25 * cells / (ms / steps / 1e3) / 1e9
    else:
        out["bb_embedded_cells"] = desc.s ** (2 * level)
        out["hbm_gbs_2B_per_embedded_cell"] = 2 * desc.s ** (2 * level) / (ms / steps / 1e3) / 1e9
    sim.close()
    torch.cuda.empty_cache()
    return out


def maps_throughput(desc, level, n=1 << 26):
    sim = Simulation(desc, level, Backend.GpuCompact, SimOptions(memory_cap=1 << 42))
    w, h = sim.compact_dims()
    side = sim.side()
    g = torch.Generator(device="cuda").manual_seed(1)
    comp = torch.stack([torch.randint(0, w, (n,), device="cuda", generator=g),
                        torch.randint(0, h, (n,), device="cuda", generator=g)], 1).to(torch.int32).contiguous()
    emb = torch.empty_like(comp)
    torch.cuda.synchronize()  # the engine runs on its own stream
    back = torch.empty_like(comp)
    res = {}
    for variant in ("digit", "mma", "tc05"):
        sim.lambda_batch_device(comp.data_ptr(), emb.data_ptr(), n, variant)  # warm
        t_l = sim.lambda_batch_device(comp.data_ptr(), emb.data_ptr(), n, variant)
        sim.nu_batch_device(emb.data_ptr(), back.data_ptr(), n, variant)
        t_n = sim.nu_batch_device(emb.data_ptr(), back.data_ptr(), n, variant)
        torch.cuda.synchronize()
        ok = bool(torch.equal(back, comp))
        res[variant] = {"lambda_maps_per_s": n / (t_l / 1e3), "nu_maps_per_s": n / (t_n / 1e3),
                        "round_trip_exact": ok}
    sim.close()
    return {"fractal": desc.name, "level": level, "coords": n, **res,
            "side": side}


def main():
    T = builtin_descriptor("sierpinski-triangle")
    Cp = builtin_descriptor("sierpinski-carpet")
    H = load_descriptor("@" + os.path.join(ROOT, "descriptors", "h-fractal.desc"))
    Y = load_descriptor("@" + os.path.join(ROOT, "descriptors", "candy.desc"))
    out = {"gpu": torch.cuda.get_device_name(0), "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
    out["config0_T_r10"] = [run(T, 10, steps=100), run(T, 10, steps=100, kernel="naive"),
                            run(T, 10, Backend.GpuBoundingBox, steps=100)]
    out["config1_T_r16"] = [run(T, 16, steps=1000), run(T, 16, steps=200, kernel="tiled"),
                            run(T, 16, steps=3, kernel="naive", maps="digit"),
                            run(T, 16, steps=3, kernel="naive", maps="mma"),
                            run(T, 16, Backend.GpuBoundingBox, steps=10)]
    out["config1_maps"] = [maps_throughput(T, 16), maps_throughput(T, 20)]
    out["config2_carpet_r9"] = [run(Cp, 9, steps=500), run(Cp, 9, steps=50, kernel="tiled"),
                                run(Cp, 9, Backend.GpuBoundingBox, steps=10)]
    out["config3_T_r18_vs_bb"] = [run(T, 18, steps=20), run(T, 18, steps=20, kernel="tiled"),
                                  run(T, 18, Backend.GpuBoundingBox, steps=3)]
    out["config3_T_r20"] = [run(T, 20, steps=100), run(T, 20, steps=20, kernel="tiled"), run(T, 22, steps=20)]
    K = FractalDescriptor("k6s3", 6, 3, [(0, 0), (1, 0), (2, 0), (0, 1), (1, 2), (2, 2)])
    jit, gen = {"NBBGPU_JIT_FORCE": "1"}, {"NBBGPU_GENERIC": "1"}
    out["config4_generic"] = [run(H, 11, steps=20), run(H, 11, steps=20, env=jit), run(H, 11, steps=20, env=gen),
                              run(Y, 9, steps=20), run(Y, 9, steps=20, env=jit), run(Y, 9, steps=20, env=gen),
                              run(K, 12, steps=20), run(K, 12, steps=20, env=gen),
                              run(H, 10, steps=20), run(Y, 8, steps=20)]
    out["bb_baseline"] = [run(Cp, 10, Backend.GpuBoundingBox, steps=3), run(Cp, 11, Backend.GpuBoundingBox, steps=2),
                          run(H, 9, Backend.GpuBoundingBox, steps=5), run(Y, 7, Backend.GpuBoundingBox, steps=5),
                          run(Cp, 10, steps=20), run(Cp, 11, steps=20)]
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
