"""GPU Simulation: host-side mirror of nbb::Simulation (proj/include/nbb/stencil.hpp:69-122)
for the two GPU backends, calling the C ABI (include/nbbgpu.h) through ctypes.

Same method names, argument meaning and error behaviour as the reference:
seed_random / step / cell / set_cell / state_hash / front / iteration, and
run_simulation (stencil.cpp:416-439).  Every state transition runs on the GPU;
there is no CPU path in this module.
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import numpy as np

from . import _abi
from .descriptor import FractalDescriptor
from .errors import OutOfDomain
from .stencil import Backend, Neighborhood, StencilRule

DEFAULT_MEMORY_CAP = 2 << 30  # kDefaultMemoryCap, proj/include/nbb/grid.hpp:13

KERNELS = {"auto": 0, "naive": 1, "tiled": 2, "packed": 3, "table": 4}
MAP_VARIANTS = {"digit": 0, "mma": 1, "tc05": 2}


@dataclass
class SimOptions:
    """SimOptions (stencil.hpp:59-64) plus the GPU selectors."""
    block_size: int = 0
    workers: int = 1
    neighbor_table: bool = False
    memory_cap: int = DEFAULT_MEMORY_CAP
    device: int = 0
    kernel: str = "auto"
    map_variant: str = "digit"
    # SimOptions::gpus (additive): > 1 -> one process drives `gpus`
    # partitions (distributed.MultiGpuSimulation) on `devices` (default 0..gpus-1)
    gpus: int = 1
    devices: Optional[List[int]] = None


@dataclass
class HostGrid:
    """front() of a GPU backend: a host mirror of Grid (grid.hpp:21-66), downloaded
    on demand and valid until the next step."""
    layout: str
    data: np.ndarray
    width: int
    height: int
    side: int

    def stored_cell_count(self) -> int:
        return int(self.data.size)

    def footprint_bytes(self) -> int:
        return int(self.data.size)


class Simulation:
    def __new__(cls, desc: FractalDescriptor = None, level: int = 0, backend: Backend = Backend.GpuCompact,
                options: Optional[SimOptions] = None):
        if cls is Simulation and options is not None and options.gpus > 1:
            from .distributed import MultiGpuSimulation
            return MultiGpuSimulation(desc, level, backend, options)
        return super().__new__(cls)

    def __init__(self, desc: FractalDescriptor, level: int,
                 backend: Backend = Backend.GpuCompact, options: Optional[SimOptions] = None):
        options = options or SimOptions()
        desc.validate()
        if backend not in (Backend.GpuCompact, Backend.GpuBoundingBox, Backend.GpuLambda):
            raise OutOfDomain(f"backend '{backend.value}' is a CPU backend of the reference; "
                              "this engine provides gpu-compact, gpu-bb and gpu-lambda")
        # option validation, stencil.cpp:128-135; neighbor_table selects the GPU
        # neighbour-table kernel (stencil.cpp:340-352, 401-414)
        if options.block_size > 0 and backend != Backend.GpuCompact:
            raise OutOfDomain("block size applies to the compact backend only")
        if options.neighbor_table and (backend != Backend.GpuCompact or options.block_size > 0):
            raise OutOfDomain("the neighbor table applies to the linear compact backend only")
        self.desc = desc
        self._level = level
        self._backend = backend
        self.options = options
        L = _abi.lib()
        h = C.c_void_p()
        if backend == Backend.GpuBoundingBox:
            mode = 1
        elif backend == Backend.GpuLambda:
            mode = 2
        else:
            mode = 3 if options.block_size > 0 else 0
        _abi.check(L.nbbgpu_create_ex(_abi.replica_array(desc.replicas), desc.replica_count,
                                      desc.growth, level, mode, int(options.block_size),
                                      options.device, int(options.memory_cap), C.byref(h)))
        self._h = h
        w, hh, side = C.c_int64(), C.c_int64(), C.c_int64()
        _abi.check(L.nbbgpu_dims(h, C.byref(w), C.byref(hh), C.byref(side)))
        self._w, self._hgt, self._side = w.value, hh.value, side.value
        kernel = options.kernel
        if options.neighbor_table and kernel == "auto":
            kernel = "table"
        if kernel != "auto":
            _abi.check(L.nbbgpu_set_kernel(h, KERNELS[kernel]))
        if options.map_variant != "digit":
            _abi.check(L.nbbgpu_set_map_variant(h, MAP_VARIANTS[options.map_variant]))
        self._front_cache: Optional[HostGrid] = None

    # -- lifetime -------------------------------------------------------------
    def close(self) -> None:
        if getattr(self, "_h", None):
            _abi.lib().nbbgpu_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- accessors (stencil.hpp:74-79) -----------------------------------------
    def backend(self) -> Backend:
        return self._backend

    def level(self) -> int:
        return self._level

    def side(self) -> int:
        return self._side

    def compact_dims(self) -> Tuple[int, int]:
        return self._w, self._hgt

    def iteration(self) -> int:
        v = C.c_int64()
        _abi.check(_abi.lib().nbbgpu_iteration(self._h, C.byref(v)))
        return v.value

    def stored_cells(self) -> int:
        v = C.c_uint64()
        _abi.check(_abi.lib().nbbgpu_stored_cells(self._h, C.byref(v)))
        return v.value

    def peak_bytes(self) -> int:
        v = C.c_uint64()
        _abi.check(_abi.lib().nbbgpu_peak_bytes(self._h, C.byref(v)))
        return v.value

    def active_kernel(self) -> Tuple[str, int]:
        k, q = C.c_int(), C.c_int()
        _abi.check(_abi.lib().nbbgpu_active_kernel(self._h, C.byref(k), C.byref(q)))
        return {1: "naive", 2: "tiled", 3: "packed", 4: "table"}[k.value], q.value

    def packed_program(self) -> Tuple[str, int]:
        """("table" | "builtin" | "jit" | "none", micro-block level) of the packed kernel."""
        prog, bl = C.c_int(), C.c_int()
        _abi.check(_abi.lib().nbbgpu_packed_program(self._h, C.byref(prog), C.byref(bl)))
        return {0: "none", 1: "table", 2: "builtin", 3: "jit"}[prog.value], bl.value

    def handle(self):
        return self._h

    # -- state ------------------------------------------------------------------
    def seed_random(self, seed: int, density: float) -> None:
        """stencil.cpp:138-180"""
        self._front_cache = None
        _abi.check(_abi.lib().nbbgpu_seed(self._h, int(seed) & (2**64 - 1), float(density)))

    def step(self, rule: StencilRule, nsteps: int = 1) -> None:
        """nsteps x Simulation::step (stencil.cpp:262-289)"""
        self._front_cache = None
        _abi.check(_abi.lib().nbbgpu_step(self._h, rule.birth & 0xFFFF, rule.survive & 0xFFFF,
                                          int(rule.neighborhood == Neighborhood.Moore), int(nsteps)))

    def step_timed(self, rule: StencilRule, nsteps: int) -> float:
        """Steps and returns the device time (ms) of the step kernels (CUDA events)."""
        self._front_cache = None
        ms = C.c_float()
        _abi.check(_abi.lib().nbbgpu_step_timed(self._h, rule.birth & 0xFFFF, rule.survive & 0xFFFF,
                                                int(rule.neighborhood == Neighborhood.Moore),
                                                int(nsteps), C.byref(ms)))
        return ms.value

    def step_profiled(self, rule: StencilRule, nsteps: int):
        """(total device ms, device ms of the main step kernels alone, engine kernel launches)."""
        self._front_cache = None
        tot, main, n = C.c_float(), C.c_float(), C.c_uint64()
        _abi.check(_abi.lib().nbbgpu_step_profiled(self._h, rule.birth & 0xFFFF, rule.survive & 0xFFFF,
                                                   int(rule.neighborhood == Neighborhood.Moore),
                                                   int(nsteps), C.byref(tot), C.byref(main), C.byref(n)))
        return tot.value, main.value, n.value

    def state_hash(self) -> int:
        """stencil.cpp:196-234"""
        v = C.c_uint64()
        _abi.check(_abi.lib().nbbgpu_state_hash(self._h, C.byref(v)))
        return v.value

    def front(self) -> HostGrid:
        if self._front_cache is None:
            n = self.stored_cells()
            buf = np.empty(n, dtype=np.uint8)
            _abi.check(_abi.lib().nbbgpu_download(self._h, buf.ctypes.data, n))
            layout = ("embedded" if self._backend in (Backend.GpuBoundingBox, Backend.GpuLambda) else
                      "blocked-compact" if self.options.block_size > 0 else "linear-compact")
            self._front_cache = HostGrid(layout, buf, self._w, self._hgt, self._side)
        return self._front_cache

    def upload(self, data: np.ndarray) -> None:
        data = np.ascontiguousarray(data, dtype=np.uint8)
        self._front_cache = None
        _abi.check(_abi.lib().nbbgpu_upload(self._h, data.ctypes.data, data.size))

    def cell(self, e) -> int:
        """stencil.cpp:182-188: e = (x, y) embedded; holes read 0."""
        v = C.c_uint8()
        _abi.check(_abi.lib().nbbgpu_get_cell(self._h, int(e[0]), int(e[1]), C.byref(v)))
        return v.value

    def set_cell(self, e, state: int) -> None:
        """stencil.cpp:190-194"""
        self._front_cache = None
        _abi.check(_abi.lib().nbbgpu_set_cell(self._h, int(e[0]), int(e[1]), int(state) & 0xFF))

    # -- batched maps (north-star item 1) ----------------------------------------
    def lambda_batch(self, coords: np.ndarray, variant: str = "digit"):
        coords = np.ascontiguousarray(coords, dtype=np.int32).reshape(-1, 2)
        out = np.empty_like(coords)
        ms = C.c_float()
        _abi.check(_abi.lib().nbbgpu_lambda_batch(self._h, MAP_VARIANTS[variant], coords.ctypes.data,
                                                  out.ctypes.data, coords.shape[0], C.byref(ms)))
        return out, ms.value

    def nu_batch(self, coords: np.ndarray, variant: str = "digit"):
        coords = np.ascontiguousarray(coords, dtype=np.int32).reshape(-1, 2)
        out = np.empty_like(coords)
        ms = C.c_float()
        _abi.check(_abi.lib().nbbgpu_nu_batch(self._h, MAP_VARIANTS[variant], coords.ctypes.data,
                                              out.ctypes.data, coords.shape[0], C.byref(ms)))
        return out, ms.value

    def lambda_batch_device(self, in_ptr: int, out_ptr: int, count: int, variant: str = "digit") -> float:
        ms = C.c_float()
        _abi.check(_abi.lib().nbbgpu_lambda_batch(self._h, MAP_VARIANTS[variant], C.c_void_p(in_ptr),
                                                  C.c_void_p(out_ptr), count, C.byref(ms)))
        return ms.value

    def nu_batch_device(self, in_ptr: int, out_ptr: int, count: int, variant: str = "digit") -> float:
        ms = C.c_float()
        _abi.check(_abi.lib().nbbgpu_nu_batch(self._h, MAP_VARIANTS[variant], C.c_void_p(in_ptr),
                                              C.c_void_p(out_ptr), count, C.byref(ms)))
        return ms.value


@dataclass
class RunResult:
    state_hash: int = 0
    steps: int = 0
    step_ms: List[float] = field(default_factory=list)
    total_ms: float = 0.0


def run_simulation(desc: FractalDescriptor, level: int, backend: Backend, rule: StencilRule,
                   steps: int, seed: int, density: float,
                   options: Optional[SimOptions] = None) -> RunResult:
    """stencil.cpp:416-439: construct, seed, time each step, return the hash."""
    if steps < 0:
        raise OutOfDomain("steps must be >= 0")
    with Simulation(desc, level, backend, options) as sim:
        sim.seed_random(seed, density)
        res = RunResult()
        t0 = time.perf_counter()
        for _ in range(steps):
            a = time.perf_counter()
            sim.step(rule)
            res.step_ms.append((time.perf_counter() - a) * 1e3)
        res.total_ms = (time.perf_counter() - t0) * 1e3
        res.steps = steps
        res.state_hash = sim.state_hash()
    return res
