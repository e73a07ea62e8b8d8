"""The reference's other two layouts on the GPU, bit-exact
against the C oracle (oracle/nbb_oracle.c, itself pinned to the reference library)
and against the reference library itself (oracle/_ref) after every step:

* gpu-lambda  -- Backend::CompactGrid (stencil.cpp:313-332): embedded storage,
                 stepped over the k^r compact indices; its bytes equal the bb ones.
* blocked     -- Backend::Compact with SimOptions::block_size (grid.cpp:54-63,
                 stencil.cpp:370-399): k^(r-m) blocks of rho x rho mini boxes.
Mirrors proj/tests/test_stencil.cpp:97-122 (layout-independent seeding),
:155-182 (randomized cross-backend equality) and :185-210 (B0 closure)."""
import numpy as np
import pytest

import oracle
from conftest import desc_from_trace
from paper_2110_12952_b200 import (Backend, SimOptions, Simulation, StencilRule, Neighborhood,
                                   builtin_descriptor, conway_rule)
from paper_2110_12952_b200.descriptor import FractalDescriptor

pytestmark = pytest.mark.gpu

T = builtin_descriptor("sierpinski-triangle")
CARPET = builtin_descriptor("sierpinski-carpet")
VICSEK = builtin_descriptor("vicsek")
H = FractalDescriptor("h", 7, 3, [(0, 0), (2, 0), (0, 1), (1, 1), (2, 1), (0, 2), (2, 2)])
Y = FractalDescriptor("y", 12, 4, [(1, 0), (2, 0), (0, 1), (1, 1), (2, 1), (3, 1), (0, 2),
                                  (1, 2), (2, 2), (3, 2), (1, 3), (2, 3)])


def _rules(rng, n):
    out = [conway_rule(), StencilRule.parse("B012345678/S012345678")]
    for i in range(n):
        out.append(StencilRule(int(rng.integers(0, 512)), int(rng.integers(0, 512)),
                               Neighborhood.Moore if i % 2 else Neighborhood.VonNeumann))
    return out


def _lockstep(desc, r, backend, mode, block_size, rule, seed, steps=4):
    o = oracle.Oracle(desc.replicas, desc.k, desc.s, r, mode=mode, block_size=block_size)
    o.seed(seed, 0.5)
    sim = Simulation(desc, r, backend, SimOptions(block_size=block_size, memory_cap=1 << 40))
    sim.seed_random(seed, 0.5)
    assert np.array_equal(sim.front().data, o.front)
    for i in range(steps):
        sim.step(rule)
        o.step(rule.birth, rule.survive, rule.moore)
        assert np.array_equal(sim.front().data, o.front), (desc.name, r, mode, block_size, rule.to_string(), i)
    assert sim.state_hash() == o.state_hash()
    sim.close()


def test_lambda_backend_vs_oracle():
    rng = np.random.default_rng(11)
    for desc, r in [(T, 5), (T, 9), (CARPET, 3), (VICSEK, 4), (H, 3), (Y, 3)]:
        for rule in _rules(rng, 2):
            _lockstep(desc, r, Backend.GpuLambda, "lambda", 0, rule, int(rng.integers(0, 2**40)))


def test_lambda_bytes_equal_bb_golden(golden):
    # compact, bb and lambda agree; lambda's buffer is bb's
    for t in golden["traces"]:
        if t["level"] > 10 or not any("bb_fnv" in v for v in t["steps"].values()):
            continue
        d = desc_from_trace(t)
        sim = Simulation(d, t["level"], Backend.GpuLambda, SimOptions(memory_cap=1 << 40))
        sim.seed_random(t["seed"], t["density"])
        rule = StencilRule(t["birth"], t["survive"],
                           Neighborhood.Moore if t["moore"] else Neighborhood.VonNeumann)
        cur = 0
        for s_ in sorted(int(k) for k in t["steps"]):
            sim.step(rule, s_ - cur)
            cur = s_
            g = t["steps"][str(s_)]
            assert f"{sim.state_hash():016x}" == g["state_hash"]
            if "bb_fnv" in g:
                assert f"{oracle.fnv1a64(sim.front().data):016x}" == g["bb_fnv"]


@pytest.mark.parametrize("desc,r,rhos", [(T, 6, (2, 4, 16)), (T, 9, (4, 16)), (CARPET, 3, (3, 9)),
                                         (VICSEK, 4, (3, 9)), (H, 3, (3,)), (Y, 3, (4, 16))])
def test_blocked_layout_vs_oracle(desc, r, rhos):
    rng = np.random.default_rng(r * 7 + desc.k)
    for rho in rhos:
        for rule in _rules(rng, 2):
            _lockstep(desc, r, Backend.GpuCompact, "blocked", rho, rule, int(rng.integers(0, 2**40)))


def test_blocked_and_lambda_vs_reference_library():
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    for desc, r, backend, mode, rho in [(T, 8, Backend.GpuCompact, "compact", 16),
                                        (CARPET, 4, Backend.GpuCompact, "compact", 9),
                                        (T, 8, Backend.GpuLambda, "lambda", 0),
                                        (VICSEK, 5, Backend.GpuLambda, "lambda", 0)]:
        ref = oracle.RefSim(desc.replicas, desc.k, desc.s, r, backend=mode, block_size=rho)
        ref.seed_random(33, 0.5)
        sim = Simulation(desc, r, backend, SimOptions(block_size=rho, memory_cap=1 << 40))
        sim.seed_random(33, 0.5)
        for i in range(5):
            assert np.array_equal(sim.front().data, ref.front()), (desc.name, mode, rho, i)
            assert sim.state_hash() == ref.state_hash()
            ref.step(0x8, 0xC, True)
            sim.step(conway_rule())


def test_seeding_is_layout_independent():
    # test_stencil.cpp:97-122: bb, lambda, linear and blocked agree cell by cell
    sims = [Simulation(CARPET, 3, b, SimOptions(block_size=bs)) for b, bs in
            [(Backend.GpuBoundingBox, 0), (Backend.GpuLambda, 0), (Backend.GpuCompact, 0),
             (Backend.GpuCompact, 3)]]
    for s_ in sims:
        s_.seed_random(1234, 0.4)
    o = oracle.Oracle(CARPET.replicas, 8, 3, 3)
    for y in range(27):
        for x in range(27):
            vals = {s_.cell((x, y)) for s_ in sims}
            assert len(vals) == 1, (x, y)
            if o.to_compact(x, y) is None:
                assert vals == {0}


def test_blocked_b0_keeps_filler_dead_and_set_cell():
    # test_stencil.cpp:185-210: filler slots stay 0 in the raw buffer under B0 rules
    rule = StencilRule.parse("B012345678/S012345678")
    sim = Simulation(T, 3, Backend.GpuCompact, SimOptions(block_size=4))
    sim.seed_random(5, 0.5)
    sim.step(rule, 3)
    o = oracle.Oracle(T.replicas, 3, 2, 3, mode="blocked", block_size=4)
    buf = sim.front().data
    for y in range(8):
        for x in range(8):
            idx = o.blocked_index(x, y)
            if idx >= 0 and (x & y):
                assert buf[idx] == 0
    sim.set_cell((1, 0), 0)
    assert sim.cell((1, 0)) == 0
    sim.set_cell((1, 0), 1)
    assert sim.cell((1, 0)) == 1
    assert sim.cell((1, 1)) == 0  # hole
