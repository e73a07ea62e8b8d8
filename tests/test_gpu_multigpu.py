"""SimOptions(gpus=N): one process drives N packed partitions with the in-process
peer-memory transport (nbbgpu_p2p_attach_local, nbbgpu_step_async).  On the test
box every "GPU" is cuda:0 (devices=[0] * N); the protocol (peer planes, pushes,
arrival counters, async enqueue) is the one N devices use.  Results must equal the
single-GPU run byte for byte (acceptance C9 across GPU counts)."""
import numpy as np
import pytest

from paper_2110_12952_b200 import (Backend, SimOptions, Simulation, StencilRule, Neighborhood,
                                   builtin_descriptor, conway_rule)
from paper_2110_12952_b200.descriptor import FractalDescriptor
from paper_2110_12952_b200.distributed import MultiGpuSimulation

pytestmark = pytest.mark.gpu

T = builtin_descriptor("sierpinski-triangle")
CARPET = builtin_descriptor("sierpinski-carpet")
H = FractalDescriptor("h", 7, 3, [(0, 0), (2, 0), (0, 1), (1, 1), (2, 1), (0, 2), (2, 2)])


def _compare(desc, level, n, rule, steps, seed=7):
    one = Simulation(desc, level, Backend.GpuCompact, SimOptions(kernel="packed", memory_cap=1 << 40))
    multi = Simulation(desc, level, Backend.GpuCompact,
                       SimOptions(gpus=n, devices=[0] * n, memory_cap=1 << 40))
    assert isinstance(multi, MultiGpuSimulation)
    one.seed_random(seed, 0.5)
    multi.seed_random(seed, 0.5)
    assert multi.state_hash() == one.state_hash()
    for k in (1, steps - 1):
        one.step(rule, k)
        multi.step(rule, k)
        assert multi.iteration() == one.iteration()
        assert multi.state_hash() == one.state_hash(), (desc.name, level, n)
        assert np.array_equal(multi.front().data, one.front().data), (desc.name, level, n)
    one.close()
    multi.close()


@pytest.mark.parametrize("fused", ["1", "0"])
@pytest.mark.parametrize("n", [2, 3, 8])
def test_multigpu_matches_single(monkeypatch, n, fused):
    # fused: the triangle B3/S23 step kernels push the peers' boundary words and
    # signal them in-kernel; "0": the separate push kernel after every step
    monkeypatch.setenv("NBBGPU_FUSED_PUSH", fused)
    _compare(T, 12, n, conway_rule(), 6)                     # q=6: in-kernel halo + counters
    _compare(T, 17, n, conway_rule(), 4)                     # q=8
    _compare(CARPET, 5, n, conway_rule(), 5)                 # halo kernel, interleaved records
    _compare(H, 6, n, StencilRule(0x49, 0x1A6, Neighborhood.VonNeumann), 4)


def test_multigpu_cells_and_upload():
    multi = Simulation(T, 9, Backend.GpuCompact, SimOptions(gpus=2, devices=[0, 0]))
    one = Simulation(T, 9, Backend.GpuCompact, SimOptions(kernel="packed"))
    for s in (one, multi):
        s.seed_random(3, 0.4)
        s.set_cell((5, 2), 1)
        s.set_cell((0, 0), 0)
        s.step(conway_rule(), 3)
    for e in [(0, 0), (5, 2), (511, 0), (3, 500), (100, 100), (511, 511)]:
        assert multi.cell(e) == one.cell(e), e
    data = one.front().data.copy()
    multi.upload(data)
    assert np.array_equal(multi.front().data, data)
    one.step(conway_rule(), 2)
    multi.step(conway_rule(), 2)
    assert multi.state_hash() == one.state_hash()
    one.close()
    multi.close()


def _ngpus():
    import torch
    return torch.cuda.device_count()


@pytest.mark.skipif(_ngpus() < 2, reason="needs two distinct GPUs")
def test_multigpu_distinct_devices():
    # kernel attributes (opt-in shared memory, 16-CTA clusters) are per device: the
    # second device's ws3 / pack kernels must launch too
    n = min(_ngpus(), 4)
    one = Simulation(T, 16, Backend.GpuCompact, SimOptions(kernel="packed", memory_cap=1 << 40))
    multi = Simulation(T, 16, Backend.GpuCompact, SimOptions(gpus=n, memory_cap=1 << 40))
    one.seed_random(42, 0.5)
    multi.seed_random(42, 0.5)
    one.step(conway_rule(), 5)
    multi.step(conway_rule(), 5)
    assert multi.state_hash() == one.state_hash()
    one.close()
    multi.close()


def test_second_handle_on_same_device_after_first():
    # a fresh handle (new tables, same kernels) still launches: attributes are keyed
    # per (kernel, device), not per process
    for level in (12, 16):
        a = Simulation(T, level, Backend.GpuCompact, SimOptions(kernel="packed"))
        a.seed_random(1, 0.5)
        a.step(conway_rule(), 3)
        b = Simulation(T, level, Backend.GpuCompact, SimOptions(kernel="packed"))
        b.seed_random(1, 0.5)
        b.step(conway_rule(), 3)
        assert a.state_hash() == b.state_hash()
        a.close()
        b.close()
