"""The C-ABI library loads and exports every symbol include/nbbgpu.h declares;
host-only planning entry points work without a GPU.  CPU only."""
import ctypes as C
import os
import re

import pytest

from paper_2110_12952_b200 import _abi
from paper_2110_12952_b200.descriptor import builtin_descriptor, load_descriptor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "nbbgpu.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(nbbgpu_[a-z_0-9]+)\s*\(", text)))


def test_header_symbols_exported():
    lib = C.CDLL(_abi.SO_PATH)
    names = declared_functions()
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # the ctypes binding covers the whole header
    assert set(names) == set(_abi.SIGNATURES), set(names) ^ set(_abi.SIGNATURES)


def test_version_and_error_channel():
    L = _abi.lib()
    assert L.nbbgpu_version() == 1
    assert L.nbbgpu_device_count() >= 0
    # invalid descriptor fails with ParseError through the status code (no GPU needed)
    rep = _abi.replica_array([(0, 0), (0, 0)])
    h = C.c_void_p()
    rc = L.nbbgpu_create(rep, 2, 2, 3, 0, 0, 1 << 30, C.byref(h))
    assert rc == 1  # NBBGPU_ERR_PARSE
    assert b"duplicate" in L.nbbgpu_last_error()


def _tiles(desc, r, q=-1, moore=1):
    info = (C.c_int32 * 8)()
    _abi.check(_abi.lib().nbbgpu_plan_tiles(_abi.replica_array(desc.replicas), desc.k, desc.s, r,
                                            q, moore, info))
    return list(info)


def test_tile_plans():
    T = builtin_descriptor("sierpinski-triangle")
    q, wq, Cc, nH, L, Wc, Hc, dmask = _tiles(T, 20)
    assert (q, wq, Cc, L) == (6, 27, 729, 14)
    assert nH == 8  # sub-triangles touch only at corners: O(1) halo per tile
    assert (Wc, Hc) == (3 ** 7, 3 ** 7)
    assert bin(dmask).count("1") == 6
    # von Neumann uses a subset of the Moore links
    assert _tiles(T, 20, moore=0)[3] <= nH
    carpet = builtin_descriptor("sierpinski-carpet")
    q, wq, Cc, nH, *_ = _tiles(carpet, 9)
    assert (q, wq, Cc) == (2, 8, 64) and nH == 40
    vicsek = builtin_descriptor("vicsek")
    assert _tiles(vicsek, 8)[:4] == [4, 25, 625, 4]


def test_tile_level_choice():
    L = _abi.lib()
    for name, r, expect in [("sierpinski-triangle", 1, 0), ("sierpinski-triangle", 3, 2),
                            ("sierpinski-triangle", 5, 4), ("sierpinski-triangle", 16, 6),
                            ("sierpinski-carpet", 1, 0), ("sierpinski-carpet", 5, 2)]:
        d = builtin_descriptor(name)
        q = C.c_int()
        _abi.check(L.nbbgpu_plan_tile_level(_abi.replica_array(d.replicas), d.k, d.s, r, C.byref(q)))
        assert q.value == expect, (name, r)


def test_partition_ranges_cover_array():
    T = builtin_descriptor("sierpinski-triangle")
    rep = _abi.replica_array(T.replicas)
    for r, n in [(12, 2), (12, 3), (16, 8), (20, 8)]:
        prev = 0
        for rank in range(n):
            lo, hi = C.c_uint64(), C.c_uint64()
            _abi.check(_abi.lib().nbbgpu_plan_partition(rep, 3, 2, r, -1, rank, n, C.byref(lo), C.byref(hi)))
            assert lo.value == prev
            prev = hi.value
        assert prev == 3 ** r


def test_jit_compiles_custom_descriptor_kernels():
    # a descriptor without built-in wiring gets the ws3 micro-block kernel compiled
    # for it at run time (NVRTC, no GPU needed); built-in descriptors do not
    L = _abi.lib()
    buf = C.create_string_buffer(512)
    custom = [((6, 3), [(0, 0), (1, 0), (2, 0), (0, 1), (1, 2), (2, 2)], 12),
              ((4, 3), [(0, 0), (2, 0), (1, 1), (0, 2)], 10),
              ((10, 4), [(0, 0), (1, 0), (2, 0), (3, 0), (0, 1), (3, 1), (0, 2), (1, 3), (2, 3), (3, 3)], 7)]
    for (k, s), reps, level in custom:
        rc = L.nbbgpu_jit_compile_check(_abi.replica_array(reps), k, s, level, 1, buf, 512)
        assert rc == 0, L.nbbgpu_last_error()
        assert b"step_packed_ws3_kernel" in buf.value and b"JitTag" in buf.value
    T = builtin_descriptor("sierpinski-triangle")
    rc = L.nbbgpu_jit_compile_check(_abi.replica_array(T.replicas), 3, 2, 12, 1, buf, 512)
    assert rc == 3 and b"run-time" in L.nbbgpu_last_error()
