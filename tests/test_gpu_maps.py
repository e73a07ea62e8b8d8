"""lambda / nu batch maps on the GPU, all three variants (CUDA-core digit loop, the
exact-integer tensor-core form on mma.sync and on tcgen05.mma kind::i8 with TMEM
accumulators), against the C oracle restatement of
CoordMapper (maps.cpp:80-146): exhaustive at small levels (acceptance C1-C3
style), random samples at the large configs."""
import numpy as np
import pytest

import oracle
from paper_2110_12952_b200 import Backend, SimOptions, Simulation, builtin_descriptor
from paper_2110_12952_b200.descriptor import FractalDescriptor

pytestmark = pytest.mark.gpu

T = builtin_descriptor("sierpinski-triangle")
CARPET = builtin_descriptor("sierpinski-carpet")
VICSEK = builtin_descriptor("vicsek")
H = FractalDescriptor("h", 7, 3, [(0, 0), (2, 0), (0, 1), (1, 1), (2, 1), (0, 2), (2, 2)])
Y = FractalDescriptor("y", 12, 4, [(1, 0), (2, 0), (0, 1), (1, 1), (2, 1), (3, 1), (0, 2),
                                  (1, 2), (2, 2), (3, 2), (1, 3), (2, 3)])


def oracle_nu(o, pts):
    out = np.full_like(pts, -1)
    for i, (x, y) in enumerate(pts):
        if 0 <= x < o.side and 0 <= y < o.side:
            c = o.to_compact(int(x), int(y))
            if c is not None:
                out[i] = c
    return out


def oracle_lambda(o, pts):
    out = np.full_like(pts, -1)
    for i, (cx, cy) in enumerate(pts):
        if 0 <= cx < o.w and 0 <= cy < o.h:
            out[i] = o.to_embedded(int(cx), int(cy))
    return out


@pytest.mark.parametrize("variant", ["digit", "mma", "tc05"])
@pytest.mark.parametrize("desc,rmax", [(T, 9), (CARPET, 4), (VICSEK, 5), (H, 4), (Y, 3)])
def test_maps_exhaustive(desc, rmax, variant):
    for r in range(rmax + 1):
        o = oracle.Oracle(desc.replicas, desc.k, desc.s, r)
        sim = Simulation(desc, r, Backend.GpuCompact)
        n = o.side
        xs, ys = np.meshgrid(np.arange(-1, n + 1), np.arange(-1, n + 1))
        emb = np.stack([xs.ravel(), ys.ravel()], axis=1).astype(np.int32)
        got, _ = sim.nu_batch(emb, variant)
        assert np.array_equal(got, oracle_nu(o, emb)), (desc.name, r, variant)
        cxs, cys = np.meshgrid(np.arange(-1, o.w + 1), np.arange(-1, o.h + 1))
        cmp_ = np.stack([cxs.ravel(), cys.ravel()], axis=1).astype(np.int32)
        got, _ = sim.lambda_batch(cmp_, variant)
        assert np.array_equal(got, oracle_lambda(o, cmp_)), (desc.name, r, variant)
        # round trip lambda(nu(e)) = e on fractal cells
        back, _ = sim.lambda_batch(sim.nu_batch(emb, variant)[0], variant)
        fr = oracle_nu(o, emb)[:, 0] >= 0
        assert np.array_equal(back[fr], emb[fr])
        sim.close()


@pytest.mark.parametrize("variant", ["digit", "mma", "tc05"])
@pytest.mark.parametrize("desc,r", [(T, 20), (T, 16), (CARPET, 9), (H, 11), (Y, 9)])
def test_maps_random_large(desc, r, variant):
    o = oracle.Oracle(desc.replicas, desc.k, desc.s, r)
    rng = np.random.default_rng(r * 31 + desc.k)
    sim = Simulation(desc, r, Backend.GpuCompact, SimOptions(memory_cap=1 << 40)) if desc.k ** r < 4e9 else None
    if sim is None:
        pytest.skip("level too large for a handle")
    m = 4000
    comp = np.stack([rng.integers(0, o.w, m), rng.integers(0, o.h, m)], axis=1).astype(np.int32)
    emb_true = oracle_lambda(o, comp)
    got, _ = sim.lambda_batch(comp, variant)
    assert np.array_equal(got, emb_true)
    # nu of fractal cells gives the compact coords back; random points mostly holes
    got, _ = sim.nu_batch(emb_true, variant)
    assert np.array_equal(got, comp)
    rnd = np.stack([rng.integers(0, o.side, m), rng.integers(0, o.side, m)], axis=1).astype(np.int32)
    got, _ = sim.nu_batch(rnd, variant)
    assert np.array_equal(got, oracle_nu(o, rnd))
    sim.close()
