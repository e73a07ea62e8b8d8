"""Run-time specialised micro-block kernels (csrc/jit.inc): descriptors with no
built-in wiring -- parsed at run time like the reference's descriptor files
(descriptor.cpp:110-162) -- get the warp-specialised micro-block step kernel
compiled for their own replica table.  Byte-exact against the oracle at every step,
for Moore / von Neumann / random / B0 rules; the built-in descriptors forced through
the same path (NBBGPU_JIT_FORCE=1) reproduce the built-in kernels' states."""
import numpy as np
import pytest

import oracle
from paper_2110_12952_b200 import (Backend, Neighborhood, SimOptions, Simulation, StencilRule,
                                   builtin_descriptor, conway_rule)
from paper_2110_12952_b200.descriptor import FractalDescriptor

pytestmark = pytest.mark.gpu

CUSTOM = [
    (FractalDescriptor("k6s3", 6, 3, [(0, 0), (1, 0), (2, 0), (0, 1), (1, 2), (2, 2)]), 8),
    (FractalDescriptor("k4s3", 4, 3, [(0, 0), (2, 0), (1, 1), (0, 2)]), 9),
    (FractalDescriptor("k5s3", 5, 3, [(0, 0), (1, 0), (1, 1), (2, 1), (1, 2)]), 8),
    (FractalDescriptor("k7s3", 7, 3, [(0, 0), (1, 0), (2, 0), (1, 1), (0, 2), (1, 2), (2, 2)]), 7),
    (FractalDescriptor("k10s4", 10, 4, [(0, 0), (1, 0), (2, 0), (3, 0), (0, 1), (3, 1), (0, 2), (1, 3),
                                        (2, 3), (3, 3)]), 6),
    (FractalDescriptor("k2s2", 2, 2, [(0, 0), (1, 1)]), 16),
    (FractalDescriptor("k13s5", 13, 5, [(0, 0), (2, 0), (4, 0), (1, 1), (3, 1), (0, 2), (2, 2), (4, 2),
                                        (1, 3), (3, 3), (0, 4), (2, 4), (4, 4)]), 5),
    (FractalDescriptor("k9s3", 9, 3, [(x, y) for y in range(3) for x in range(3)]), 6),
    # k = 8 row blocks (BW % 4 == 0): interleaved record words (rec_word, padded records)
    (FractalDescriptor("k8s3c", 8, 3, [(x, y) for y in range(3) for x in range(3) if (x, y) != (0, 0)]), 6),
]


def _lockstep(desc, level, rule, seed, steps):
    o = oracle.Oracle(desc.replicas, desc.k, desc.s, level)
    o.seed(seed, 0.5)
    sim = Simulation(desc, level, Backend.GpuCompact, SimOptions(kernel="packed", memory_cap=1 << 40))
    sim.seed_random(seed, 0.5)
    prog = sim.packed_program()
    for i in range(steps):
        o.step(rule.birth, rule.survive, rule.moore)
        sim.step(rule)
        assert np.array_equal(sim.front().data, o.front), (desc.name, level, rule.to_string(), i)
    assert sim.state_hash() == o.state_hash()
    sim.close()
    return prog


@pytest.mark.parametrize("case", range(len(CUSTOM)))
def test_custom_descriptor_runs_jit_kernel(case):
    desc, level = CUSTOM[case]
    desc.validate()
    rng = np.random.default_rng(31 + case)
    rules = [conway_rule(), StencilRule(0x48, 0x1C, Neighborhood.VonNeumann),
             StencilRule(int(rng.integers(0, 512)), int(rng.integers(0, 512)), Neighborhood.Moore),
             StencilRule(int(rng.integers(0, 512)) | 1, int(rng.integers(0, 512)), Neighborhood.Moore)]  # B0
    for i, rule in enumerate(rules):
        prog, bl = _lockstep(desc, level, rule, 100 + i, 4)
        assert prog == "jit" and bl in (1, 2), (desc.name, prog)


@pytest.mark.parametrize("name,level", [("h", 9), ("candy", 6), ("carpet", 7), ("vicsek", 8), ("triangle", 13)])
def test_builtin_descriptors_through_jit_match(monkeypatch, name, level):
    desc = {"h": FractalDescriptor("h", 7, 3, [(0, 0), (2, 0), (0, 1), (1, 1), (2, 1), (0, 2), (2, 2)]),
            "candy": FractalDescriptor("candy", 12, 4, [(1, 0), (2, 0), (0, 1), (1, 1), (2, 1), (3, 1), (0, 2),
                                                        (1, 2), (2, 2), (3, 2), (1, 3), (2, 3)]),
            "carpet": builtin_descriptor("sierpinski-carpet"), "vicsek": builtin_descriptor("vicsek"),
            "triangle": builtin_descriptor("sierpinski-triangle")}[name]
    sims = {}
    for force in ("0", "1"):
        monkeypatch.setenv("NBBGPU_JIT_FORCE", force)
        s = Simulation(desc, level, Backend.GpuCompact, SimOptions(kernel="packed", memory_cap=1 << 40))
        s.seed_random(9, 0.5)
        sims[force] = s
    assert sims["1"].packed_program()[0] == "jit"
    for rule in (conway_rule(), StencilRule(0x49, 0x1A6, Neighborhood.VonNeumann)):
        for s in sims.values():
            s.step(rule, 3)
        assert sims["0"].state_hash() == sims["1"].state_hash()
        assert np.array_equal(sims["0"].front().data, sims["1"].front().data)
    for s in sims.values():
        s.close()


@pytest.mark.parametrize("ilv", ["0", "1"])
@pytest.mark.parametrize("name,level", [("k6s3", 11), ("carpet", 10), ("h", 10)])
def test_jit_many_groups_match_table_program(monkeypatch, name, level, ilv):
    # >= 2048 groups: the run-time specialised kernel with its bt warps, compile-time
    # stage size and the register-form transposed gather (halo_bt_regs_kernel) == the
    # table-driven program (NBBGPU_GENERIC=1, B plane + direct gather), across a rule
    # switch, a set_cell and odd / even call lengths; with interleaved records
    # (NBBGPU_JIT_ILV=1: rec_word, padded records) and without
    monkeypatch.setenv("NBBGPU_JIT_ILV", ilv)
    desc = {"k6s3": CUSTOM[0][0], "carpet": builtin_descriptor("sierpinski-carpet"),
            "h": FractalDescriptor("h", 7, 3, [(0, 0), (2, 0), (0, 1), (1, 1), (2, 1), (0, 2), (2, 2)])}[name]
    sims = {}
    for env in (("NBBGPU_JIT_FORCE", "1"), ("NBBGPU_GENERIC", "1")):
        monkeypatch.delenv("NBBGPU_JIT_FORCE", raising=False)
        monkeypatch.delenv("NBBGPU_GENERIC", raising=False)
        monkeypatch.setenv(*env)
        s = Simulation(desc, level, Backend.GpuCompact, SimOptions(kernel="packed", memory_cap=1 << 40))
        s.seed_random(17, 0.5)
        sims[env[0]] = s
    assert sims["NBBGPU_JIT_FORCE"].packed_program()[0] == "jit"
    assert sims["NBBGPU_GENERIC"].packed_program()[0] != "jit"
    vn = StencilRule(0x49, 0x1A6, Neighborhood.VonNeumann)
    for rule, n in ((conway_rule(), 3), (vn, 2), ("set", 0), (conway_rule(), 4)):
        for s in sims.values():
            if rule == "set":
                s.set_cell((0, 0), 1 - s.cell((0, 0)))
            else:
                s.step(rule, n)
        assert sims["NBBGPU_JIT_FORCE"].state_hash() == sims["NBBGPU_GENERIC"].state_hash(), (name, rule)
    for s in sims.values():
        s.close()
