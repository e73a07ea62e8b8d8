"""Device-side output and lockstep verification: the PBM of
proj/tests/test_pbm.cpp:10-52 rendered on the GPU from every layout, the embedded
view against the C oracle, and verify_stencil (oracle.cpp:132-186) over the GPU
bb / lambda / compact backends, including a deliberately corrupted run."""
import io

import numpy as np
import pytest

import oracle
from paper_2110_12952_b200 import (Backend, CapacityError, SimOptions, Simulation, StencilRule,
                                   builtin_descriptor, conway_rule, embedded_view, render_pbm,
                                   verify_stencil, write_pbm)

pytestmark = pytest.mark.gpu
T = builtin_descriptor("sierpinski-triangle")
CARPET = builtin_descriptor("sierpinski-carpet")


def test_pbm_known_answers():
    # test_pbm.cpp:13-27
    sim = Simulation(T, 1, Backend.GpuCompact)
    sim.seed_random(0, 1.0)
    out = io.BytesIO()
    write_pbm(sim, out)
    assert out.getvalue() == b"P1\n2 2\n11\n10\n"
    sim.seed_random(0, 0.0)
    assert render_pbm(sim) == b"P1\n2 2\n00\n00\n"


def test_pbm_identical_across_layouts():
    # test_pbm.cpp:27-42, over every GPU layout (bb, lambda, packed, tiled bytes, blocked)
    rule = conway_rule()
    sims = [Simulation(T, 9, Backend.GpuBoundingBox), Simulation(T, 9, Backend.GpuLambda),
            Simulation(T, 9, Backend.GpuCompact, SimOptions(kernel="packed")),
            Simulation(T, 9, Backend.GpuCompact, SimOptions(kernel="tiled")),
            Simulation(T, 9, Backend.GpuCompact, SimOptions(block_size=16))]
    for s in sims:
        s.seed_random(3, 0.5)
        s.step(rule, 8)
    pbms = [render_pbm(s) for s in sims]
    assert all(p == pbms[0] for p in pbms)
    assert pbms[0][:11] == b"P1\n512 512\n"
    # against the oracle's embedded view
    o = oracle.Oracle(T.replicas, 3, 2, 9, mode="bb")
    o.seed(3, 0.5)
    o.step(8, 12, True, nsteps=8)
    rows = o.front.reshape(512, 512)
    expect = b"P1\n512 512\n" + b"".join(bytes((48 + v for v in row)) + b"\n" for row in rows)
    assert pbms[0] == expect
    assert np.array_equal(embedded_view(sims[2]), rows)


def test_pbm_render_cap_and_path(tmp_path):
    # test_pbm.cpp:43-52
    sim = Simulation(T, 6, Backend.GpuCompact)
    with pytest.raises(CapacityError):
        write_pbm(sim, io.BytesIO(), 32)
    small = Simulation(T, 1, Backend.GpuCompact)
    with pytest.raises(CapacityError):
        write_pbm(small, "/nonexistent-dir/frame.pbm")
    p = tmp_path / "f.pbm"
    write_pbm(small, str(p))
    assert p.read_bytes().startswith(b"P1\n2 2\n")


def test_verify_stencil_gpu_backends():
    rep = verify_stencil(T, 8, conway_rule(), 42, 0.5, 10)
    assert rep.passed and rep.cells_checked == 11 * 3 ** 8, rep.summary()
    rep = verify_stencil(CARPET, 4, StencilRule.parse("B36/S23"), 7, 0.4, 6)
    assert rep.passed, rep.summary()


def test_verify_stencil_detects_divergence():
    # a LockstepHook that corrupts the compact backend after iteration 2
    def corrupt(it, sims):
        if it == 2:
            comp = sims[2]
            for x in range(comp.side()):
                try:
                    comp.set_cell((x, 0), 1 - comp.cell((x, 0)))
                    return
                except Exception:
                    continue
    rep = verify_stencil(T, 6, conway_rule(), 1, 0.5, 5, post_step=corrupt)
    assert not rep.passed
    assert "gpu-compact diverges from bb at iteration 2" in rep.violations[0]
