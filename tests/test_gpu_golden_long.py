"""Every BASELINE config pinned to the reference at its horizon, through every kernel
family: tests/golden/golden_long.json holds state hashes of the UNMODIFIED reference
(oracle/_ref, tests/golden/make_golden_long.py) for T r=16 to step 1000, carpet r=9
to step 500, T r=18 / r=20 to step 10, H r=10/11 and Candy r=8/9 (config 5's
~1e9-cell custom fractals).  test_gpu_parity.test_large_levels_hash steps the
default (micro-block packed) path; here the generic transition-table program
(step_packed_kernel, NBBGPU_GENERIC=1), the tiled byte kernel, and the paper's
per-cell kernel with CUDA-core and tensor-core maps reach the same hashes."""
import os

import pytest

from conftest import desc_from_trace
from paper_2110_12952_b200 import Backend, SimOptions, Simulation, StencilRule, Neighborhood

pytestmark = pytest.mark.gpu


def _rule(t):
    return StencilRule(t["birth"], t["survive"], Neighborhood.Moore if t["moore"] else Neighborhood.VonNeumann)


def _walk(t, kernel="auto", maps="digit", env=None, upto=None, monkeypatch=None):
    if env and monkeypatch is not None:
        for k, v in env.items():
            monkeypatch.setenv(k, v)
    d = desc_from_trace(t)
    sim = Simulation(d, t["level"], Backend.GpuCompact,
                     SimOptions(kernel=kernel, map_variant=maps, memory_cap=1 << 42))
    sim.seed_random(t["seed"], t["density"])
    rule = _rule(t)
    cur = 0
    checked = []
    for s in sorted(int(k) for k in t["state_hash"]):
        if upto is not None and s > upto:
            break
        sim.step(rule, s - cur)
        cur = s
        got = f"{sim.state_hash():016x}"
        assert got == t["state_hash"][str(s)], (t["fractal"], t["level"], kernel, maps, env, s)
        checked.append(s)
    kern = sim.active_kernel()
    sim.close()
    return checked, kern


@pytest.mark.parametrize("key", ["t16", "c9", "t18", "h10", "y8", "h11", "y9", "t20"])
def test_generic_transition_table_path(golden_long, key, monkeypatch):
    # BASELINE configs[4] names "the generic transition-table path": the packed
    # program built from the parsed descriptor alone, no compile-time wiring
    if key not in golden_long:
        pytest.skip(f"{key} not in golden_long.json")
    checked, kern = _walk(golden_long[key], kernel="packed", env={"NBBGPU_GENERIC": "1"}, monkeypatch=monkeypatch)
    assert kern[0] == "packed" and len(checked) >= 2


@pytest.mark.parametrize("key", ["t16", "c9", "t18", "h10", "h11", "t20"])
def test_tiled_byte_kernel(golden_long, key):
    if key not in golden_long:
        pytest.skip(f"{key} not in golden_long.json")
    checked, kern = _walk(golden_long[key], kernel="tiled", upto=100)
    assert kern[0] == "tiled" and len(checked) >= 2


@pytest.mark.parametrize("maps", ["digit", "mma"])
def test_paper_per_cell_kernel_t16(golden_long, maps):
    # BASELINE configs[1]: T r=16 with the lambda / nu maps on CUDA cores and on the
    # tensor cores (mma.sync u8), the paper's one-thread-per-cell kernel
    checked, kern = _walk(golden_long["t16"], kernel="naive", maps=maps, upto=10)
    assert kern[0] == "naive" and checked == [0, 1, 3, 10]


@pytest.mark.parametrize("key", ["c9", "t18", "h10", "y8", "h11", "y9", "t20"])
def test_run_time_specialised_kernel(golden_long, key, monkeypatch):
    # the descriptor's micro-block wiring compiled at run time (jit.inc) -- the path
    # every custom descriptor takes -- forced onto the BASELINE configs
    if key not in golden_long:
        pytest.skip(f"{key} not in golden_long.json")
    monkeypatch.setenv("NBBGPU_JIT_FORCE", "1")
    t = golden_long[key]
    sim = Simulation(desc_from_trace(t), t["level"], Backend.GpuCompact,
                     SimOptions(kernel="packed", memory_cap=1 << 42))
    assert sim.packed_program()[0] == "jit"
    sim.close()
    checked, kern = _walk(t, kernel="packed")
    assert len(checked) >= 2
