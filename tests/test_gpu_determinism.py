"""Long lockstep runs of the multi-set warp-specialised kernels at full size.

The ws3 step kernel's consumer warps form NGRP group sets sharing one TMA stage ring;
with NS not a multiple of NGRP a set could pass a stage's parity wait one phase early
when TMA loads completed out of order, corrupting one warp's slice of one group about
once per 10^4 group-steps (found by tools/divergence.py on the run-time kernel of a
K(n,6,3) descriptor at r=12: NGRP 3, NS 7).  Here the run-time kernel (NGRP 3) and
the Vicsek kernel (NGRP 16) step ~5e6 group-steps in lockstep with the table-driven
program (one set, __syncthreads per group), hashes compared every 25 steps."""
import pytest

from paper_2110_12952_b200 import Backend, SimOptions, Simulation, builtin_descriptor, conway_rule
from paper_2110_12952_b200.descriptor import FractalDescriptor

pytestmark = pytest.mark.gpu

K63 = FractalDescriptor("k6s3", 6, 3, [(0, 0), (1, 0), (2, 0), (0, 1), (1, 2), (2, 2)])


def _sim(desc, level, monkeypatch, **env):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    s = Simulation(desc, level, Backend.GpuCompact, SimOptions(kernel="packed", memory_cap=1 << 42))
    for k in env:
        monkeypatch.delenv(k)
    s.seed_random(42, 0.5)
    return s


@pytest.mark.parametrize("name,level,steps", [("k6s3", 12, 100), ("vicsek", 12, 300)])
def test_multiset_kernel_lockstep(monkeypatch, name, level, steps):
    desc = K63 if name == "k6s3" else builtin_descriptor("vicsek")
    a = _sim(desc, level, monkeypatch)
    r = _sim(desc, level, monkeypatch, NBBGPU_GENERIC="1", NBBGPU_JIT="0")
    assert a.packed_program()[0] in ("jit", "builtin") and r.packed_program()[0] == "table"
    rule = conway_rule()
    for i in range(0, steps, 25):
        a.step(rule, 25)
        r.step(rule, 25)
        assert a.state_hash() == r.state_hash(), (name, level, i + 25)
    a.close()
    r.close()
