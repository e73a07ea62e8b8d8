"""Partitioned GPU path on ONE GPU: N handles play N ranks (owned tile rows,
tiled kernel restricted to them, device pack/unpack of the halo bytes); the
transport between "ranks" is a device-to-device copy instead of NCCL.  After
every step the summed owned hashes and the owned bytes equal an unpartitioned
run (acceptance C9 across GPU counts)."""
import ctypes as C

import numpy as np
import pytest
import torch

from paper_2110_12952_b200 import (Backend, SimOptions, Simulation, StencilRule, Neighborhood,
                                   builtin_descriptor, _abi)
from paper_2110_12952_b200.distributed import PartitionPlan, wrap_u64_sum

pytestmark = pytest.mark.gpu


def _run(desc, level, nranks, rule, steps, kernel="auto"):
    L = _abi.lib()
    full = Simulation(desc, level, Backend.GpuCompact, SimOptions(kernel=kernel, memory_cap=1 << 40))
    full.seed_random(5, 0.5)
    ranks = []
    for r in range(nranks):
        sim = Simulation(desc, level, Backend.GpuCompact, SimOptions(kernel=kernel, memory_cap=1 << 40))
        sim.seed_random(5, 0.5)
        _abi.check(L.nbbgpu_partition(sim.handle(), r, nranks))
        kern, q = sim.active_kernel()
        if kern == "packed":
            plan = PartitionPlan(desc, level, r, nranks, tile_level=q, packed=True)
        else:
            plan = PartitionPlan(desc, level, r, nranks, tile_level=-1 if kernel == "tiled" else 0)
        for p in plan.peers:
            s = plan.send[p]
            _abi.check(L.nbbgpu_halo_set_sends(sim.handle(), p, s.ctypes.data if s.size else None, s.size))
        ranks.append((sim, plan))
    for step in range(steps):
        full.step(rule)
        for sim, _ in ranks:
            sim.step(rule)
        packed = {}
        for r, (sim, plan) in enumerate(ranks):
            for p in plan.peers:
                n = int(plan.send[p].size)
                buf = torch.empty(max(1, n), dtype=torch.int32 if plan.packed else torch.uint8,
                                  device="cuda")
                _abi.check(L.nbbgpu_halo_pack(sim.handle(), p, C.c_void_p(buf.data_ptr())))
                packed[(r, p)] = buf
        for r, (sim, plan) in enumerate(ranks):
            for p in plan.peers:
                if plan.recv[p].size:
                    buf = packed[(p, r)]
                    assert buf.numel() >= plan.recv[p].size
                    _abi.check(L.nbbgpu_halo_unpack(sim.handle(), p, C.c_void_p(buf.data_ptr())))
        parts = []
        ref = full.front().data
        for sim, plan in ranks:
            v = C.c_uint64()
            _abi.check(L.nbbgpu_state_hash_owned(sim.handle(), C.byref(v)))
            parts.append(v.value)
            got = sim.front().data
            m = plan.owned_cell_mask()
            assert np.array_equal(got[m], ref[m]), (desc.name, level, step)
        assert wrap_u64_sum(parts) == full.state_hash(), (desc.name, level, step)


@pytest.mark.parametrize("nranks", [2, 3, 8])
def test_partitioned_triangle(nranks):
    T = builtin_descriptor("sierpinski-triangle")
    _run(T, 12, nranks, StencilRule(8, 12, Neighborhood.Moore), 5, kernel="tiled")
    _run(T, 9, nranks, StencilRule(0x1C8, 0x6, Neighborhood.VonNeumann), 4, kernel="tiled")


def test_partitioned_other_fractals():
    C8 = builtin_descriptor("sierpinski-carpet")
    V = builtin_descriptor("vicsek")
    _run(C8, 5, 3, StencilRule(8, 12, Neighborhood.Moore), 4, kernel="tiled")
    _run(V, 6, 2, StencilRule(0x6, 0x9, Neighborhood.Moore), 4, kernel="tiled")


def test_partitioned_naive_kernel():
    T = builtin_descriptor("sierpinski-triangle")
    _run(T, 8, 3, StencilRule(8, 12, Neighborhood.Moore), 4, kernel="naive")


@pytest.mark.parametrize("nranks", [2, 3, 8])
def test_partitioned_packed(nranks):
    T = builtin_descriptor("sierpinski-triangle")
    C8 = builtin_descriptor("sierpinski-carpet")
    _run(T, 12, nranks, StencilRule(8, 12, Neighborhood.Moore), 5, kernel="packed")
    _run(T, 9, nranks, StencilRule(0x1C9, 0x6, Neighborhood.VonNeumann), 4, kernel="packed")
    _run(C8, 5, nranks, StencilRule(8, 12, Neighborhood.Moore), 4, kernel="packed")


@pytest.mark.parametrize("hw", ["0", "1"])
def test_partitioned_packed_q8_halo_warps(monkeypatch, hw):
    # T q=8 partitions: halo words gathered in the step kernel (hw=1) or by the halo kernel
    monkeypatch.setenv("NBBGPU_PACKED_Q", "8")
    monkeypatch.setenv("NBBGPU_HALO_WARPS", hw)
    T = builtin_descriptor("sierpinski-triangle")
    for n in (2, 3, 8):
        _run(T, 14, n, StencilRule(8, 12, Neighborhood.Moore), 4, kernel="packed")
