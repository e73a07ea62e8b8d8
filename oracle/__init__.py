"""ctypes bindings for the parity checkers.  TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline / reference
arm import this package.  The product (``paper_2110_12952_b200``) never does.

* ``liboracle.so``   -- nbb_oracle.c, a plain-C restatement of the reference path
  (every function cites the reference file:line it follows).
* ``_ref/libnbbref.so`` -- the unmodified reference library compiled from
  /root/reference/proj/src by oracle/Makefile, behind ref_shim.cpp.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_ORACLE_SO = os.path.join(HERE, "liboracle.so")
_REF_SO = os.path.join(HERE, "_ref", "libnbbref.so")

MAX_LEVEL = 40
MAX_S = 16


def build(quiet: bool = True) -> None:
    """make -C oracle (C restatement always; reference lib when /root/reference exists)."""
    out = subprocess.run(["make", "-C", HERE, "-j8"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


class _Mapper(C.Structure):
    _fields_ = [
        ("k", C.c_int), ("s", C.c_int), ("r", C.c_int),
        ("side", C.c_int64), ("w", C.c_int64), ("h", C.c_int64),
        ("spow", C.c_int64 * (MAX_LEVEL + 1)),
        ("id_of_subbox", C.c_int16 * (MAX_S * MAX_S)),
        ("rep_gx", C.c_int32 * (MAX_S * MAX_S)),
        ("rep_gy", C.c_int32 * (MAX_S * MAX_S)),
        ("stride_x", C.c_int64 * MAX_LEVEL),
        ("stride_y", C.c_int64 * MAX_LEVEL),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_ORACLE_SO):
            build()
        L = C.CDLL(_ORACLE_SO)
        P = C.POINTER
        L.nbbo_mapper_init.argtypes = [P(_Mapper), P(C.c_int32), C.c_int, C.c_int, C.c_int]
        L.nbbo_mapper_init.restype = C.c_int
        L.nbbo_try_to_compact.argtypes = [P(_Mapper), C.c_int64, C.c_int64, P(C.c_int64), P(C.c_int64)]
        L.nbbo_try_to_compact.restype = C.c_int
        L.nbbo_to_compact_via_mma.argtypes = L.nbbo_try_to_compact.argtypes
        L.nbbo_to_compact_via_mma.restype = C.c_int
        L.nbbo_to_embedded.argtypes = [P(_Mapper), C.c_int64, C.c_int64, P(C.c_int64), P(C.c_int64)]
        L.nbbo_to_embedded.restype = None
        L.nbbo_splitmix64.argtypes = [C.c_uint64]
        L.nbbo_splitmix64.restype = C.c_uint64
        L.nbbo_cell_alive.argtypes = [C.c_uint64, C.c_int64, C.c_int64, C.c_double]
        L.nbbo_cell_alive.restype = C.c_int
        L.nbbo_coord_mix.argtypes = [C.c_int64, C.c_int64]
        L.nbbo_coord_mix.restype = C.c_uint64
        L.nbbo_seed.argtypes = [P(_Mapper), C.c_int, C.c_uint64, C.c_double, C.c_void_p]
        L.nbbo_seed.restype = None
        L.nbbo_state_hash.argtypes = [P(_Mapper), C.c_int, C.c_void_p]
        L.nbbo_state_hash.restype = C.c_uint64
        L.nbbo_state_hash_range.argtypes = [P(_Mapper), C.c_void_p, C.c_int64, C.c_int64]
        L.nbbo_state_hash_range.restype = C.c_uint64
        L.nbbo_step_compact.argtypes = [P(_Mapper), C.c_uint16, C.c_uint16, C.c_int, C.c_void_p,
                                        C.c_void_p, C.c_int64, C.c_int64]
        L.nbbo_step_compact.restype = None
        L.nbbo_step.argtypes = [P(_Mapper), C.c_int, C.c_uint16, C.c_uint16, C.c_int, C.c_void_p,
                                C.c_void_p, C.c_int]
        L.nbbo_step.restype = None
        L.nbbo_fnv1a64.argtypes = [C.c_void_p, C.c_int64]
        L.nbbo_fnv1a64.restype = C.c_uint64
        L.nbbo_blocked_index.argtypes = [P(_Mapper), P(_Mapper), C.c_int64, C.c_int64, C.c_int64]
        L.nbbo_blocked_index.restype = C.c_int64
        L.nbbo_blocked_seed.argtypes = [P(_Mapper), P(_Mapper), C.c_int64, C.c_uint64, C.c_double, C.c_void_p]
        L.nbbo_blocked_seed.restype = None
        L.nbbo_blocked_hash.argtypes = [P(_Mapper), P(_Mapper), C.c_int64, C.c_void_p]
        L.nbbo_blocked_hash.restype = C.c_uint64
        L.nbbo_blocked_step.argtypes = [P(_Mapper), P(_Mapper), C.c_int64, C.c_uint16, C.c_uint16, C.c_int,
                                        C.c_void_p, C.c_void_p, C.c_int64, C.c_int64]
        L.nbbo_blocked_step.restype = None
        _lib = L
    return _lib


def fnv1a64(buf: np.ndarray) -> int:
    buf = np.ascontiguousarray(buf, dtype=np.uint8)
    return int(lib().nbbo_fnv1a64(buf.ctypes.data, buf.size))


class Oracle:
    """The C restatement for one (descriptor, level): maps, seeding, steps, hash.

    mode "compact" keeps the reference's linear compact buffer (cy*w+cx, k^r bytes);
    mode "bb" keeps the embedded n*n buffer; mode "lambda" (the CompactGrid
    backend) the embedded buffer stepped over the compact indices; mode "blocked"
    (block_size rho = s^m) the BlockedCompact layout of k^(r-m) rho x rho blocks.
    """

    def __init__(self, replicas, k: int, s: int, level: int, mode: str = "compact",
                 block_size: int = 0):
        self.m = _Mapper()
        arr = (C.c_int32 * (2 * k))(*[int(v) for xy in replicas for v in xy])
        if lib().nbbo_mapper_init(C.byref(self.m), arr, k, s, level) != 0:
            raise ValueError("invalid descriptor/level for the oracle")
        self.mode = {"compact": 0, "bb": 1, "lambda": 2, "blocked": 3}[mode]
        self.k, self.s, self.level = k, s, level
        self.side, self.w, self.h = self.m.side, self.m.w, self.m.h
        self.rho = 0
        if self.mode == 3:
            mexp, p = 0, 1
            while p < block_size:
                p *= s
                mexp += 1
            if p != block_size or mexp > level:
                raise ValueError("block size must be s^m with m <= level")
            self.rho = block_size
            self.mc = _Mapper()
            if lib().nbbo_mapper_init(C.byref(self.mc), arr, k, s, level - mexp) != 0:
                raise ValueError("invalid coarse level for the oracle")
            n = self.mc.w * self.mc.h * block_size * block_size
        else:
            n = self.side * self.side if self.mode in (1, 2) else self.w * self.h
        self.front = np.zeros(n, dtype=np.uint8)
        self.back = np.zeros(n, dtype=np.uint8)

    # maps ------------------------------------------------------------------
    def to_compact(self, x: int, y: int):
        cx, cy = C.c_int64(), C.c_int64()
        if not lib().nbbo_try_to_compact(C.byref(self.m), x, y, C.byref(cx), C.byref(cy)):
            return None
        return cx.value, cy.value

    def to_compact_via_mma(self, x: int, y: int):
        cx, cy = C.c_int64(), C.c_int64()
        if not lib().nbbo_to_compact_via_mma(C.byref(self.m), x, y, C.byref(cx), C.byref(cy)):
            return None
        return cx.value, cy.value

    def to_embedded(self, cx: int, cy: int):
        x, y = C.c_int64(), C.c_int64()
        lib().nbbo_to_embedded(C.byref(self.m), cx, cy, C.byref(x), C.byref(y))
        return x.value, y.value

    # simulation --------------------------------------------------------------
    def seed(self, seed: int, density: float) -> None:
        self.front[:] = 0
        self.back[:] = 0
        if self.mode == 3:
            lib().nbbo_blocked_seed(C.byref(self.m), C.byref(self.mc), self.rho, seed, density,
                                    self.front.ctypes.data)
            return
        lib().nbbo_seed(C.byref(self.m), self.mode, seed, density, self.front.ctypes.data)

    def blocked_index(self, x: int, y: int) -> int:
        return int(lib().nbbo_blocked_index(C.byref(self.m), C.byref(self.mc), self.rho, x, y))

    def step(self, birth: int = 0x8, survive: int = 0xC, moore: bool = True, nsteps: int = 1,
             threads: int = 0) -> None:
        threads = threads or min(os.cpu_count() or 1, 64)
        if self.mode == 3:
            for _ in range(nsteps):
                lib().nbbo_blocked_step(C.byref(self.m), C.byref(self.mc), self.rho, birth, survive,
                                        int(moore), self.front.ctypes.data, self.back.ctypes.data, 0,
                                        self.mc.w * self.mc.h)
                self.front, self.back = self.back, self.front
            return
        for _ in range(nsteps):
            lib().nbbo_step(C.byref(self.m), self.mode, birth, survive, int(moore),
                            self.front.ctypes.data, self.back.ctypes.data, threads)
            self.front, self.back = self.back, self.front

    def step_range(self, birth, survive, moore, i0, i1) -> None:
        """Compact step over [i0, i1) into the back buffer (no swap)."""
        lib().nbbo_step_compact(C.byref(self.m), birth, survive, int(moore),
                                self.front.ctypes.data, self.back.ctypes.data, i0, i1)

    def swap(self) -> None:
        self.front, self.back = self.back, self.front

    def state_hash(self) -> int:
        if self.mode == 3:
            return int(lib().nbbo_blocked_hash(C.byref(self.m), C.byref(self.mc), self.rho,
                                               self.front.ctypes.data))
        return int(lib().nbbo_state_hash(C.byref(self.m), self.mode, self.front.ctypes.data))

    def state_hash_range(self, i0: int, i1: int) -> int:
        return int(lib().nbbo_state_hash_range(C.byref(self.m), self.front.ctypes.data, i0, i1))

    def fnv(self) -> int:
        return fnv1a64(self.front)


# --------------------------------------------------------------------------
# The reference itself (oracle/_ref/libnbbref.so)
# --------------------------------------------------------------------------
_ref = None


def ref_available() -> bool:
    return os.path.exists(_REF_SO)


def ref_lib():
    global _ref
    if _ref is None:
        if not os.path.exists(_REF_SO):
            raise FileNotFoundError(_REF_SO + " (run make -C oracle where /root/reference exists)")
        L = C.CDLL(_REF_SO)
        P = C.POINTER
        L.nbbref_last_error.restype = C.c_char_p
        L.nbbref_create.argtypes = [P(C.c_int32), C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                    C.c_int, C.c_int, C.c_uint64, P(C.c_void_p)]
        L.nbbref_create_builtin.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                            C.c_uint64, P(C.c_void_p)]
        L.nbbref_destroy.argtypes = [C.c_void_p]
        L.nbbref_seed.argtypes = [C.c_void_p, C.c_uint64, C.c_double]
        L.nbbref_step.argtypes = [C.c_void_p, C.c_uint16, C.c_uint16, C.c_int, C.c_int64]
        L.nbbref_state_hash.argtypes = [C.c_void_p]
        L.nbbref_state_hash.restype = C.c_uint64
        L.nbbref_front.argtypes = [C.c_void_p, P(C.c_void_p)]
        L.nbbref_front.restype = C.c_int64
        L.nbbref_cell.argtypes = [C.c_void_p, C.c_int64, C.c_int64, P(C.c_uint8)]
        L.nbbref_set_cell.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_uint8]
        L.nbbref_to_compact.argtypes = [P(C.c_int32), C.c_int, C.c_int, C.c_int, C.c_int64, C.c_int64,
                                        P(C.c_int64), P(C.c_int64)]
        L.nbbref_to_embedded.argtypes = L.nbbref_to_compact.argtypes
        L.nbbref_parallel_seed.argtypes = [C.c_void_p, C.c_uint64, C.c_double, C.c_int]
        L.nbbref_parallel_seed_range.argtypes = [C.c_void_p, C.c_uint64, C.c_double, C.c_int64,
                                                 C.c_int64, C.c_int]
        L.nbbref_sample_step.argtypes = [C.c_void_p, C.c_uint16, C.c_uint16, C.c_int, C.c_int64,
                                         C.c_int64, C.c_int]
        _ref = L
    return _ref


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _check(code):
    if code != 0:
        raise RefError(code, ref_lib().nbbref_last_error().decode())


BACKENDS = {"bb": 0, "lambda": 1, "compact": 2}


class RefSim:
    """nbb::Simulation from the unmodified reference sources."""

    def __init__(self, replicas, k, s, level, backend="compact", block_size=0, workers=1,
                 neighbor_table=False, memory_cap=1 << 40):
        L = ref_lib()
        h = C.c_void_p()
        arr = (C.c_int32 * (2 * k))(*[int(v) for xy in replicas for v in xy])
        _check(L.nbbref_create(arr, k, s, level, BACKENDS[backend], block_size, workers,
                               int(neighbor_table), memory_cap, C.byref(h)))
        self.h = h
        self.k, self.s, self.level = k, s, level

    def __del__(self):
        if getattr(self, "h", None):
            ref_lib().nbbref_destroy(self.h)
            self.h = None

    def seed_random(self, seed, density):
        _check(ref_lib().nbbref_seed(self.h, seed, density))

    def parallel_seed(self, seed, density, workers):
        _check(ref_lib().nbbref_parallel_seed(self.h, seed, density, workers))

    def step(self, birth=0x8, survive=0xC, moore=True, nsteps=1):
        _check(ref_lib().nbbref_step(self.h, birth, survive, int(moore), nsteps))

    def parallel_seed_range(self, seed, density, i0, i1, workers):
        _check(ref_lib().nbbref_parallel_seed_range(self.h, seed, density, i0, i1, workers))

    def sample_step(self, birth, survive, moore, i0, i1, workers):
        _check(ref_lib().nbbref_sample_step(self.h, birth, survive, int(moore), i0, i1, workers))

    def state_hash(self) -> int:
        return int(ref_lib().nbbref_state_hash(self.h))

    def front(self) -> np.ndarray:
        p = C.c_void_p()
        n = ref_lib().nbbref_front(self.h, C.byref(p))
        buf = (C.c_uint8 * n).from_address(p.value)
        return np.frombuffer(buf, dtype=np.uint8).copy()

    def cell(self, x, y) -> int:
        v = C.c_uint8()
        _check(ref_lib().nbbref_cell(self.h, x, y, C.byref(v)))
        return v.value

    def set_cell(self, x, y, v):
        _check(ref_lib().nbbref_set_cell(self.h, x, y, v))


def ref_to_compact(replicas, k, s, level, x, y):
    arr = (C.c_int32 * (2 * k))(*[int(v) for xy in replicas for v in xy])
    cx, cy = C.c_int64(), C.c_int64()
    _check(ref_lib().nbbref_to_compact(arr, k, s, level, x, y, C.byref(cx), C.byref(cy)))
    return cx.value, cy.value


def ref_to_embedded(replicas, k, s, level, cx, cy):
    arr = (C.c_int32 * (2 * k))(*[int(v) for xy in replicas for v in xy])
    x, y = C.c_int64(), C.c_int64()
    _check(ref_lib().nbbref_to_embedded(arr, k, s, level, cx, cy, C.byref(x), C.byref(y)))
    return x.value, y.value
