"""Parity at BASELINE.json's full sizes through size-independent properties: the
oracle cannot step 3^20 cells in test time, so independent GPU kernels (packed
bit-sliced, tiled byte layout, the paper's per-cell naive kernel) must agree with
each other step after step at T r=20 and r=22, and the reference's own r=20
golden hashes (steps 0, 1) pin the start.  Conversions are checked
by an upload/download round trip of the full r=20 state."""
import numpy as np
import pytest

import oracle
from paper_2110_12952_b200 import (Backend, SimOptions, Simulation, StencilRule, Neighborhood,
                                   builtin_descriptor, conway_rule)

pytestmark = pytest.mark.gpu
T = builtin_descriptor("sierpinski-triangle")


def _sim(level, kernel):
    s = Simulation(T, level, Backend.GpuCompact, SimOptions(kernel=kernel, memory_cap=1 << 42))
    s.seed_random(42, 0.5)
    return s


def test_r20_packed_tiled_naive_agree():
    p, t = _sim(20, "packed"), _sim(20, "tiled")
    assert f"{p.state_hash():016x}" == "b97b1b7132951b93"  # reference golden, step 0
    rule = conway_rule()
    for n in (1, 4, 7):
        p.step(rule, n)
        t.step(rule, n)
        if n == 1:
            assert f"{p.state_hash():016x}" == "4cc6771ca85cba3d"  # reference golden, step 1
        assert p.state_hash() == t.state_hash()
    fp = oracle.fnv1a64(p.front().data)
    p._front_cache = None
    ft = oracle.fnv1a64(t.front().data)
    assert fp == ft
    t.close()
    # the paper's per-cell kernel, two steps from the same seed
    nv = _sim(20, "naive")
    p2 = _sim(20, "packed")
    vn = StencilRule(0x48, 0x1C, Neighborhood.VonNeumann)
    for r_ in (rule, vn):
        nv.step(r_)
        p2.step(r_)
        assert nv.state_hash() == p2.state_hash()
    nv.close()
    p.close()
    p2.close()


def test_r20_upload_download_round_trip():
    p = _sim(20, "packed")
    p.step(conway_rule(), 3)
    h = p.state_hash()
    buf = p.front().data.copy()
    q = Simulation(T, 20, Backend.GpuCompact, SimOptions(kernel="packed", memory_cap=1 << 42))
    q.upload(buf)
    assert q.state_hash() == h
    del buf
    p.step(conway_rule(), 2)
    q.step(conway_rule(), 2)
    assert p.state_hash() == q.state_hash()


def test_r22_packed_matches_tiled():
    # 3^22 = 3.1e10 cells: 7.8 GB packed, 62.8 GB for the tiled byte double buffer
    p, t = _sim(22, "packed"), _sim(22, "tiled")
    assert p.state_hash() == t.state_hash()
    for _ in range(3):
        p.step(conway_rule())
        t.step(conway_rule())
        assert p.state_hash() == t.state_hash()
    t.close()
    p.close()


@pytest.mark.parametrize("case", ["h11", "c10", "y9"])
def test_large_configs_kernel_agreement(monkeypatch, case):
    # BASELINE configs 3 and 5 at full size: the packed micro-block kernel with its
    # default large-halo path (transposed boundary plane: 4-chunk transposes +
    # entry-list gather for >= 8192 groups) against the tiled byte-layout kernel
    from paper_2110_12952_b200.descriptor import FractalDescriptor
    desc, level = {
        "h11": (FractalDescriptor("h", 7, 3, [(0, 0), (2, 0), (0, 1), (1, 1), (2, 1), (0, 2), (2, 2)]), 11),
        "c10": (builtin_descriptor("sierpinski-carpet"), 10),
        "y9": (FractalDescriptor("y", 12, 4, [(1, 0), (2, 0), (0, 1), (1, 1), (2, 1), (3, 1), (0, 2),
                                              (1, 2), (2, 2), (3, 2), (1, 3), (2, 3)]), 9),
    }[case]
    sims = {}
    for k in ("packed", "tiled"):
        s = Simulation(desc, level, Backend.GpuCompact, SimOptions(kernel=k, memory_cap=1 << 42))
        s.seed_random(42, 0.5)
        sims[k] = s
    for n in (1, 3):
        for rule in (conway_rule(), StencilRule(0x49, 0x1A6, Neighborhood.VonNeumann)):
            for s in sims.values():
                s.step(rule, n)
            assert sims["packed"].state_hash() == sims["tiled"].state_hash(), (case, n)
    for s in sims.values():
        s.close()


@pytest.mark.parametrize("case", ["h11", "c10", "k12"])
def test_long_calls_graphs_and_wide_halos_agree(monkeypatch, case):
    # many steps per call at full size: the >= 8192-group wide-halo gather, the bt
    # warps' transposed plane and the captured-graph replay (forced) against the
    # tiled byte kernel and against stream launches, with a rule switch mid-run
    from paper_2110_12952_b200.descriptor import FractalDescriptor
    desc, level = {
        "h11": (FractalDescriptor("h", 7, 3, [(0, 0), (2, 0), (0, 1), (1, 1), (2, 1), (0, 2), (2, 2)]), 11),
        "c10": (builtin_descriptor("sierpinski-carpet"), 10),
        "k12": (FractalDescriptor("k6s3", 6, 3, [(0, 0), (1, 0), (2, 0), (0, 1), (1, 2), (2, 2)]), 11),
    }[case]
    hashes = {}
    ref = "naive" if case == "k12" else "tiled"  # (no tiled-kernel tile width for k = 6)
    for label, kernel, graphs in (("tiled", ref, "0"), ("stream", "packed", "0"), ("graphs", "packed", "1")):
        monkeypatch.setenv("NBBGPU_GRAPHS", graphs)
        s = Simulation(desc, level, Backend.GpuCompact, SimOptions(kernel=kernel, memory_cap=1 << 42))
        s.seed_random(5, 0.5)
        s.step(conway_rule(), 19)
        s.step(StencilRule(0x49, 0x1A6, Neighborhood.VonNeumann), 10)
        hashes[label] = s.state_hash()
        s.close()
    assert hashes["stream"] == hashes["tiled"] == hashes["graphs"], (case, hashes)
