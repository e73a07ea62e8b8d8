"""Pins the C restatement (oracle/nbb_oracle.c) before it is trusted as the checker.

1. against the golden vectors produced by the unmodified reference
   (tests/golden/golden.json, tests/golden/make_golden.py);
2. against the reference's own known-answer tests (proj/tests/test_maps.cpp,
   test_stencil.cpp, test_grid.cpp) restated here with their file:line;
3. directly against oracle/_ref (the reference library) when it is present.
CPU only.
"""
import numpy as np
import pytest

import oracle
from conftest import desc_from_trace
from paper_2110_12952_b200.descriptor import builtin_descriptor

T = builtin_descriptor("sierpinski-triangle")
CARPET = builtin_descriptor("sierpinski-carpet")
VICSEK = builtin_descriptor("vicsek")


def O(desc, r, mode="compact"):
    return oracle.Oracle(desc.replicas, desc.k, desc.s, r, mode)


def test_map_kats():
    # proj/tests/test_maps.cpp:58-73
    assert O(T, 2).to_compact(0, 0) == (0, 0)
    assert O(T, 2).to_compact(0, 3) == (2, 2)
    assert O(T, 3).to_compact(5, 2) == (4, 2)
    assert O(CARPET, 1).to_compact(2, 1) == (4, 0)
    assert O(T, 2).to_compact(2, 2) is None          # NotInFractal
    assert O(T, 3).to_embedded(4, 2) == (5, 2)
    assert O(T, 2).to_embedded(2, 2) == (0, 3)
    assert O(T, 0).to_embedded(0, 0) == (0, 0)


def test_dims_kats():
    # proj/tests/test_maps.cpp:40-47
    assert (O(T, 0).w, O(T, 0).h) == (1, 1)
    assert (O(T, 3).w, O(T, 3).h) == (9, 3)
    assert (O(CARPET, 2).w, O(CARPET, 2).h) == (8, 8)


@pytest.mark.parametrize("desc,rmax", [(T, 7), (CARPET, 4), (VICSEK, 4)])
def test_bijection_and_mma_form(desc, rmax):
    # acceptance.cpp:62-115 (C1) and :153-174 (C3) at small levels
    for r in range(rmax + 1):
        o = O(desc, r)
        hits = np.zeros(o.w * o.h, dtype=np.int32)
        for y in range(o.side):
            for x in range(o.side):
                c = o.to_compact(x, y)
                if c is None:
                    continue
                hits[c[1] * o.w + c[0]] += 1
                assert o.to_embedded(*c) == (x, y)
                assert o.to_compact_via_mma(x, y) == c
        assert (hits == 1).all()


def test_seed_and_hash_kats():
    # test_stencil.cpp:114-121: density 0 -> hash 0; density 1 -> all alive
    o = O(CARPET, 2)
    o.seed(7, 0.0)
    assert o.state_hash() == 0
    o.seed(7, 1.0)
    assert int(o.front.sum()) == 64


def test_blinker_on_solid_grid():
    # test_stencil.cpp:69-95
    from paper_2110_12952_b200.descriptor import FractalDescriptor
    solid = FractalDescriptor("solid", 4, 2, [(0, 0), (1, 0), (0, 1), (1, 1)])
    o = O(solid, 2)
    o.seed(0, 0.0)

    def put(x, y):
        cx, cy = o.to_compact(x, y)
        o.front[cy * o.w + cx] = 1

    def get(x, y):
        cx, cy = o.to_compact(x, y)
        return int(o.front[cy * o.w + cx])

    for y in range(3):
        put(1, y)
    o.step(8, 12, True)
    assert (get(0, 1), get(1, 1), get(2, 1), get(1, 0), get(1, 2)) == (1, 1, 1, 0, 0)
    o.step(8, 12, True)
    assert (get(1, 0), get(1, 2), get(3, 0), get(3, 3)) == (1, 1, 0, 0)


def _check_trace(t, mode):
    d = desc_from_trace(t)
    o = O(d, t["level"], "bb" if mode == "bb" else "compact")
    o.seed(t["seed"], t["density"])
    steps = sorted(int(s) for s in t["steps"])
    cur = 0
    for s in steps:
        if s > cur:
            o.step(t["birth"], t["survive"], t["moore"], nsteps=s - cur)
            cur = s
        g = t["steps"][str(s)]
        assert f"{o.state_hash():016x}" == g["state_hash"], (t["fractal"], t["level"], s)
        key = "bb_fnv" if mode == "bb" else "fnv"
        if key in g:
            assert f"{o.fnv():016x}" == g[key], (t["fractal"], t["level"], s, mode)
    for s, hexbytes in t.get("dumps" if mode != "bb" else "bb_dumps", {}).items():
        pass  # dumps are checked step-by-step in the GPU tests


def test_oracle_matches_golden_traces(golden):
    for t in golden["traces"]:
        if t["level"] > 14:
            continue
        _check_trace(t, "compact")
        if t["level"] <= 10 and any("bb_fnv" in v for v in t["steps"].values()):
            _check_trace(t, "bb")


def test_oracle_matches_golden_random_trials(golden):
    for t in golden["random_c5"] + golden["random_xbackend"]:
        _check_trace(t, "compact")
        _check_trace(t, "bb")


def test_oracle_dumps_bytes(golden):
    t = golden["traces"][0]  # T r=6, dumps at steps 0,1,2,3,10
    d = desc_from_trace(t)
    o = O(d, t["level"])
    o.seed(t["seed"], t["density"])
    cur = 0
    for s in sorted(int(k) for k in t["dumps"]):
        o.step(t["birth"], t["survive"], t["moore"], nsteps=s - cur)
        cur = s
        assert o.front.tobytes().hex() == t["dumps"][str(s)]


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built (needs /root/reference)")
def test_oracle_equals_reference_directly():
    # seeded + stepped state bytes equal the reference's own buffers
    from paper_2110_12952_b200.descriptor import load_descriptor
    import os
    H = load_descriptor("@" + os.path.join(os.path.dirname(__file__), "..", "descriptors", "h-fractal.desc"))
    for desc, r in [(T, 8), (CARPET, 4), (VICSEK, 5), (H, 4)]:
        ref = oracle.RefSim(desc.replicas, desc.k, desc.s, r, backend="compact")
        ref.seed_random(5, 0.4)
        o = O(desc, r)
        o.seed(5, 0.4)
        for step in range(5):
            assert np.array_equal(ref.front(), o.front)
            assert ref.state_hash() == o.state_hash()
            ref.step(0x48, 0x1C, step % 2 == 0)
            o.step(0x48, 0x1C, step % 2 == 0)
        for (x, y) in [(0, 0), (1, 0), (3, 2)]:
            if x < o.side and y < o.side:
                c = o.to_compact(x, y)
                if c is not None:
                    assert oracle.ref_to_compact(desc.replicas, desc.k, desc.s, r, x, y) == c


def test_oracle_lambda_and_blocked_match_reference_library():
    # the C restatement of step_compact_grid (stencil.cpp:313-332) and of the blocked
    # layout (grid.cpp:54-63, stencil.cpp:161-177/217-231/370-399) against the
    # unmodified reference, byte for byte, after every step
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    T = [(0, 0), (1, 0), (0, 1)]
    C8 = [(0, 0), (1, 0), (2, 0), (0, 1), (2, 1), (0, 2), (1, 2), (2, 2)]
    V = [(1, 0), (0, 1), (1, 1), (2, 1), (1, 2)]
    for rep, k, s, r in [(T, 3, 2, 6), (C8, 8, 3, 3), (V, 5, 3, 4), (T, 3, 2, 8)]:
        for mode, bs in [("lambda", 0), ("blocked", s), ("blocked", s * s)]:
            o = oracle.Oracle(rep, k, s, r, mode=mode, block_size=bs)
            o.seed(9, 0.5)
            R = oracle.RefSim(rep, k, s, r, backend="lambda" if mode == "lambda" else "compact",
                              block_size=bs)
            R.seed_random(9, 0.5)
            assert np.array_equal(o.front, R.front()), (mode, bs)
            for i in range(5):
                birth, surv, moore = (8, 12, True) if i % 2 == 0 else (0x49, 0x1A7, False)
                o.step(birth, surv, moore)
                R.step(birth, surv, moore)
                assert np.array_equal(o.front, R.front()), (mode, bs, r, i)
                assert o.state_hash() == R.state_hash()
