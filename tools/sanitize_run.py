"""Small runs of every hot kernel family for compute-sanitizer (racecheck, synccheck,
memcheck, initcheck).  Each case runs a few steps at a small level and checks the
final hash against a second run of the same steps on the byte-layout tiled kernel.

    compute-sanitizer --tool racecheck python tools/sanitize_run.py ws3_halo_kernel

Cases: see CASES below; `all` runs every case in one process.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2110_12952_b200 import Backend, SimOptions, Simulation, builtin_descriptor, conway_rule  # noqa: E402
from paper_2110_12952_b200.descriptor import FractalDescriptor  # noqa: E402

T = builtin_descriptor("sierpinski-triangle")
C = builtin_descriptor("sierpinski-carpet")
H = FractalDescriptor("h", 7, 3, [(0, 0), (2, 0), (0, 1), (1, 1), (2, 1), (0, 2), (2, 2)])
Y = FractalDescriptor("y", 12, 4, [(1, 0), (2, 0), (0, 1), (1, 1), (2, 1), (3, 1), (0, 2), (1, 2), (2, 2),
                                   (3, 2), (1, 3), (2, 3)])
K63 = FractalDescriptor("k63", 6, 3, [(0, 0), (1, 0), (2, 0), (0, 1), (1, 2), (2, 2)])

# name: (descriptor, level, backend, kernel, env, gpus)
CASES = {
    "ws3_halo_warps": (T, 16, Backend.GpuCompact, "packed", {"NBBGPU_HALO_WARPS": "1"}, 1),
    "ws3_halo_kernel": (T, 16, Backend.GpuCompact, "packed", {"NBBGPU_HALO_WARPS": "0"}, 1),
    "resident": (T, 10, Backend.GpuCompact, "packed", {}, 1),
    "cluster8": (T, 12, Backend.GpuCompact, "packed", {}, 1),
    "cluster16": (T, 13, Backend.GpuCompact, "packed", {}, 1),
    "carpet_pws": (C, 6, Backend.GpuCompact, "packed", {}, 1),
    "h_bt": (H, 7, Backend.GpuCompact, "packed", {}, 1),
    "h_bt_warps": (H, 6, Backend.GpuCompact, "packed", {"NBBGPU_HALO_BT": "1"}, 1),
    "carpet_bt_warps": (C, 6, Backend.GpuCompact, "packed", {"NBBGPU_HALO_BT": "1"}, 1),
    "graphs": (T, 12, Backend.GpuCompact, "tiled", {}, 1),
    "candy_split": (Y, 5, Backend.GpuCompact, "packed", {}, 1),
    "jit": (K63, 6, Backend.GpuCompact, "packed", {}, 1),
    "jit_split": (Y, 5, Backend.GpuCompact, "packed", {"NBBGPU_JIT_FORCE": "1"}, 1),
    "generic": (K63, 6, Backend.GpuCompact, "packed", {"NBBGPU_GENERIC": "1"}, 1),
    "generic_h": (H, 6, Backend.GpuCompact, "packed", {"NBBGPU_GENERIC": "1"}, 1),
    "tiled": (T, 12, Backend.GpuCompact, "tiled", {}, 1),
    "naive": (T, 10, Backend.GpuCompact, "naive", {}, 1),
    "table": (T, 10, Backend.GpuCompact, "table", {}, 1),
    "bb_s2": (T, 9, Backend.GpuBoundingBox, "auto", {}, 1),
    "bb_s3": (C, 5, Backend.GpuBoundingBox, "auto", {}, 1),
    "bb_s4": (Y, 4, Backend.GpuBoundingBox, "auto", {}, 1),
    "push_p2p": (T, 12, Backend.GpuCompact, "packed", {}, 2),
    "push_p2p_q8": (T, 17, Backend.GpuCompact, "packed", {}, 2),
    # >= 2048 groups: the register-form Bt halo gather (halo_bt_regs_kernel), run-time
    # and built-in wiring; carpet / H: immediate stage addressing + bt warps
    "jit_k11": (K63, 11, Backend.GpuCompact, "packed", {}, 1),
    "carpet_c10": (C, 10, Backend.GpuCompact, "packed", {}, 1),
    "h_h10": (H, 10, Backend.GpuCompact, "packed", {}, 1),
}
BIG = {"jit_k11", "carpet_c10", "h_h10"}  # no naive-kernel reference under the sanitizer (too slow)


def run(name, steps=3):
    if name == "graphs":
        steps = 20  # > 8 steps: captured CUDA graph replay
    desc, level, backend, kernel, env, gpus = CASES[name]
    saved = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        opts = SimOptions(kernel=kernel, memory_cap=1 << 40)
        if gpus > 1:
            opts = SimOptions(gpus=gpus, devices=[0] * gpus, memory_cap=1 << 40)
        sim = Simulation(desc, level, backend, opts)
        sim.seed_random(5, 0.5)
        rule = conway_rule()
        sim.step(rule, steps)
        got = sim.state_hash()
        sim.close()
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    if name in BIG:
        print(f"{name}: ran {got:016x}", flush=True)
        return True
    # state_hash is layout independent (stencil.cpp:196-234): every case is checked
    # against the per-cell naive compact kernel
    ref = Simulation(desc, level, Backend.GpuCompact, SimOptions(kernel="naive", memory_cap=1 << 40))
    ref.seed_random(5, 0.5)
    ref.step(rule, steps)
    want = ref.state_hash()
    ref.close()
    status = "ok" if got == want else "MISMATCH"
    print(f"{name}: {status} {got:016x}", flush=True)
    return got == want


def run_maps():
    """the three map variants (digit, mma.sync, tcgen05) against each other"""
    import numpy as np
    sim = Simulation(T, 12, Backend.GpuCompact, SimOptions())
    rng = np.random.default_rng(3)
    pts = np.stack([rng.integers(0, 4096, 3000), rng.integers(0, 4096, 3000)], 1).astype(np.int32)
    outs = [sim.nu_batch(pts, v)[0] for v in ("digit", "mma", "tc05")]
    comp = np.stack([rng.integers(0, 729, 3000), rng.integers(0, 729, 3000)], 1).astype(np.int32)
    outl = [sim.lambda_batch(comp, v)[0] for v in ("digit", "mma", "tc05")]
    sim.close()
    ok = all(np.array_equal(outs[0], o) for o in outs) and all(np.array_equal(outl[0], o) for o in outl)
    print(f"maps: {'ok' if ok else 'MISMATCH'}", flush=True)
    return ok


if __name__ == "__main__":
    names = sys.argv[1:] or ["all"]
    if names == ["all"]:
        names = list(CASES) + ["maps"]
    ok = all([run_maps() if n == "maps" else run(n) for n in names])
    sys.exit(0 if ok else 1)
