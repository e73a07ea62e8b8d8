"""Device-side output and lockstep verification.

write_pbm mirrors proj/src/pbm.cpp:9-35 (plain PBM "P1", '1' = alive, render cap,
CapacityError on an unwritable path); the rows are rendered on the GPU from any
layout (nbbgpu_render_pbm) instead of n^2 host-side Simulation::cell calls.

verify_stencil mirrors proj/src/oracle.cpp:132-186: the three backends (here the
GPU bounding box, the GPU lambda backend and the GPU compact backend) step in
lockstep from the same seed and their embedded views must agree on every cell
after every iteration; the comparison runs on the device.
"""
from __future__ import annotations

import ctypes as C
import io
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Union

import numpy as np

from . import _abi
from .descriptor import FractalDescriptor
from .errors import CapacityError
from .simulation import SimOptions, Simulation
from .stencil import Backend, StencilRule

DEFAULT_RENDER_CAP = 1 << 14  # kDefaultRenderCap, proj/include/nbb/pbm.hpp:11


def render_pbm(sim: Simulation, render_cap: int = DEFAULT_RENDER_CAP) -> bytes:
    """The PBM bytes of sim's front state (pbm.cpp:9-23), rendered on the device."""
    L, n = _abi.lib(), C.c_uint64()
    _abi.check(L.nbbgpu_render_pbm(sim.handle(), None, 0, int(render_cap), C.byref(n)))
    buf = (C.c_char * n.value)()
    _abi.check(L.nbbgpu_render_pbm(sim.handle(), buf, n.value, int(render_cap), C.byref(n)))
    return bytes(buf)


def write_pbm(sim: Simulation, out: Union[str, io.IOBase], render_cap: int = DEFAULT_RENDER_CAP) -> None:
    """write_pbm(sim, stream | path, render_cap) -- pbm.cpp:9-35."""
    data = render_pbm(sim, render_cap)
    if isinstance(out, str):
        try:
            with open(out, "wb") as fh:
                fh.write(data)
        except OSError as e:
            raise CapacityError(f"cannot open '{out}' for writing") from e
        return
    try:
        out.write(data)
    except TypeError:  # text stream
        out.write(data.decode("ascii"))


def embedded_view(sim: Simulation, device_out=None) -> Optional[np.ndarray]:
    """Simulation::cell for every (x, y) as an n x n uint8 array, computed on the GPU.
    With device_out (a CUDA tensor of n*n uint8) the view stays on the device."""
    n = sim.side()
    L = _abi.lib()
    if device_out is not None:
        _abi.check(L.nbbgpu_embedded_view(sim.handle(), C.c_void_p(device_out.data_ptr()), n * n))
        return None
    out = np.empty(n * n, dtype=np.uint8)
    _abi.check(L.nbbgpu_embedded_view(sim.handle(), out.ctypes.data, n * n))
    return out.reshape(n, n)


@dataclass
class VerifyReport:
    """oracle.hpp:28-33"""
    passed: bool = True
    cells_checked: int = 0
    violations: List[str] = field(default_factory=list)

    def summary(self) -> str:
        return (("PASS" if self.passed else "FAIL") + f": {self.cells_checked} cells checked"
                + (f", {len(self.violations)} violation(s)" if self.violations else ""))


LockstepHook = Callable[[int, List[Simulation]], None]


def verify_stencil(desc: FractalDescriptor, level: int, rule: StencilRule, seed: int, density: float,
                   steps: int, post_step: Optional[LockstepHook] = None,
                   options: Optional[SimOptions] = None) -> VerifyReport:
    """oracle.cpp:132-186 on the GPU backends: bb is the reference, lambda and compact
    must agree with it on every fractal cell after every iteration."""
    import torch
    opts = options or SimOptions(memory_cap=1 << 40)
    report = VerifyReport()

    def note(msg: str) -> None:
        report.passed = False
        if len(report.violations) < 100:
            report.violations.append(msg)

    sims = [Simulation(desc, level, b, opts) for b in
            (Backend.GpuBoundingBox, Backend.GpuLambda, Backend.GpuCompact)]
    for s in sims:
        s.seed_random(seed, density)
    n = sims[0].side()
    dev = torch.device("cuda", opts.device)
    views = [torch.empty(n * n, dtype=torch.uint8, device=dev) for _ in sims]
    cells = desc.k ** level

    def compare(iteration: int) -> bool:
        for s, v in zip(sims, views):
            embedded_view(s, v)
        for s, v in zip(sims[1:], views[1:]):
            diff = torch.nonzero(v != views[0])
            if diff.numel():
                i = int(diff[0, 0])
                note(f"backend {s.backend().value} diverges from bb at iteration {iteration}, "
                     f"cell ({i % n},{i // n})")
                return False
        report.cells_checked += cells
        return True

    try:
        if not compare(0):
            return report
        for it in range(1, steps + 1):
            for s in sims:
                s.step(rule)
            if post_step is not None:
                post_step(it, sims)
            if not compare(it):
                return report
        return report
    finally:
        for s in sims:
            s.close()
