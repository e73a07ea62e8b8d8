"""ctypes binding of the C ABI (include/nbbgpu.h) -> libnbbgpu.so.

The library is built in-tree (paper_2110_12952_b200/build.py).  There is no
fallback: if the .so is missing or fails to load, every GPU entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os

from .errors import STATUS_TO_ERROR, NbbError

HERE = os.path.dirname(os.path.abspath(__file__))
# NBBGPU_LIB (A/B measurements only): another build of the same library
SO_PATH = os.environ.get("NBBGPU_LIB") or os.path.join(HERE, "libnbbgpu.so")

# name -> (restype, argtypes); mirrors include/nbbgpu.h
_P = C.POINTER
_H = C.c_void_p
SIGNATURES = {
    "nbbgpu_last_error": (C.c_char_p, []),
    "nbbgpu_version": (C.c_int, []),
    "nbbgpu_device_count": (C.c_int, []),
    "nbbgpu_create": (C.c_int, [_P(C.c_int32), C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                C.c_uint64, _P(_H)]),
    "nbbgpu_create_ex": (C.c_int, [_P(C.c_int32), C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                   C.c_uint64, _P(_H)]),
    "nbbgpu_destroy": (C.c_int, [_H]),
    "nbbgpu_seed": (C.c_int, [_H, C.c_uint64, C.c_double]),
    "nbbgpu_step": (C.c_int, [_H, C.c_uint16, C.c_uint16, C.c_int, C.c_int64]),
    "nbbgpu_step_timed": (C.c_int, [_H, C.c_uint16, C.c_uint16, C.c_int, C.c_int64, _P(C.c_float)]),
    "nbbgpu_step_profiled": (C.c_int, [_H, C.c_uint16, C.c_uint16, C.c_int, C.c_int64, _P(C.c_float),
                                       _P(C.c_float), _P(C.c_uint64)]),
    "nbbgpu_launch_count": (C.c_int, [_H, _P(C.c_uint64)]),
    "nbbgpu_state_hash": (C.c_int, [_H, _P(C.c_uint64)]),
    "nbbgpu_iteration": (C.c_int, [_H, _P(C.c_int64)]),
    "nbbgpu_stored_cells": (C.c_int, [_H, _P(C.c_uint64)]),
    "nbbgpu_dims": (C.c_int, [_H, _P(C.c_int64), _P(C.c_int64), _P(C.c_int64)]),
    "nbbgpu_download": (C.c_int, [_H, C.c_void_p, C.c_uint64]),
    "nbbgpu_upload": (C.c_int, [_H, C.c_void_p, C.c_uint64]),
    "nbbgpu_get_cell": (C.c_int, [_H, C.c_int64, C.c_int64, _P(C.c_uint8)]),
    "nbbgpu_set_cell": (C.c_int, [_H, C.c_int64, C.c_int64, C.c_uint8]),
    "nbbgpu_peak_bytes": (C.c_int, [_H, _P(C.c_uint64)]),
    "nbbgpu_embedded_view": (C.c_int, [_H, C.c_void_p, C.c_uint64]),
    "nbbgpu_render_pbm": (C.c_int, [_H, C.c_void_p, C.c_uint64, C.c_int64, _P(C.c_uint64)]),
    "nbbgpu_set_kernel": (C.c_int, [_H, C.c_int]),
    "nbbgpu_set_map_variant": (C.c_int, [_H, C.c_int]),
    "nbbgpu_active_kernel": (C.c_int, [_H, _P(C.c_int), _P(C.c_int)]),
    "nbbgpu_stream": (C.c_int, [_H, _P(C.c_void_p)]),
    "nbbgpu_packed_program": (C.c_int, [_H, _P(C.c_int), _P(C.c_int)]),
    "nbbgpu_jit_compile_check": (C.c_int, [_P(C.c_int32), C.c_int, C.c_int, C.c_int, C.c_int, C.c_char_p,
                                           C.c_uint64]),
    "nbbgpu_lambda_batch": (C.c_int, [_H, C.c_int, C.c_void_p, C.c_void_p, C.c_int64, _P(C.c_float)]),
    "nbbgpu_nu_batch": (C.c_int, [_H, C.c_int, C.c_void_p, C.c_void_p, C.c_int64, _P(C.c_float)]),
    "nbbgpu_partition": (C.c_int, [_H, C.c_int, C.c_int]),
    "nbbgpu_owned_range": (C.c_int, [_H, _P(C.c_uint64), _P(C.c_uint64)]),
    "nbbgpu_halo_needs": (C.c_int, [_H, C.c_int, C.c_void_p, _P(C.c_uint64)]),
    "nbbgpu_halo_set_sends": (C.c_int, [_H, C.c_int, C.c_void_p, C.c_uint64]),
    "nbbgpu_halo_pack": (C.c_int, [_H, C.c_int, C.c_void_p]),
    "nbbgpu_halo_unpack": (C.c_int, [_H, C.c_int, C.c_void_p]),
    "nbbgpu_state_hash_owned": (C.c_int, [_H, _P(C.c_uint64)]),
    "nbbgpu_front_device_ptr": (C.c_int, [_H, _P(C.c_void_p)]),
    "nbbgpu_nccl_unique_id": (C.c_int, [C.c_void_p, C.c_int]),
    "nbbgpu_comm_init": (C.c_int, [_H, C.c_void_p, C.c_int]),
    "nbbgpu_plan_tile_level": (C.c_int, [_P(C.c_int32), C.c_int, C.c_int, C.c_int, _P(C.c_int)]),
    "nbbgpu_plan_partition": (C.c_int, [_P(C.c_int32), C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                        C.c_int, _P(C.c_uint64), _P(C.c_uint64)]),
    "nbbgpu_plan_needs": (C.c_int, [_P(C.c_int32), C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                    C.c_int, C.c_int, C.c_void_p, _P(C.c_uint64)]),
    "nbbgpu_plan_tiles": (C.c_int, [_P(C.c_int32), C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                    _P(C.c_int32)]),
    "nbbgpu_halo_elem_bytes": (C.c_int, [_H, _P(C.c_int)]),
    "nbbgpu_p2p_handle_bytes": (C.c_int, []),
    "nbbgpu_p2p_export": (C.c_int, [_H, C.c_void_p, C.c_int]),
    "nbbgpu_p2p_attach": (C.c_int, [_H, C.c_void_p, C.c_int, C.c_int]),
    "nbbgpu_p2p_attach_local": (C.c_int, [C.c_void_p, C.c_int]),
    "nbbgpu_step_async": (C.c_int, [_H, C.c_uint16, C.c_uint16, C.c_int, C.c_int64]),
    "nbbgpu_synchronize": (C.c_int, [_H]),
    "nbbgpu_plan_packed_level": (C.c_int, [_P(C.c_int32), C.c_int, C.c_int, C.c_int, _P(C.c_int)]),
    "nbbgpu_plan_packed": (C.c_int, [_P(C.c_int32), C.c_int, C.c_int, C.c_int, C.c_int, _P(C.c_int64)]),
    "nbbgpu_plan_packed_partition": (C.c_int, [_P(C.c_int32), C.c_int, C.c_int, C.c_int, C.c_int,
                                               C.c_int, C.c_int, _P(C.c_int64), _P(C.c_int64)]),
    "nbbgpu_plan_packed_needs": (C.c_int, [_P(C.c_int32), C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                           C.c_int, C.c_int, C.c_void_p, _P(C.c_uint64)]),
    "nbbgpu_plan_packed_elem_cells": (C.c_int, [_P(C.c_int32), C.c_int, C.c_int, C.c_int, C.c_int,
                                                C.c_void_p, C.c_uint64, C.c_void_p, _P(C.c_uint64)]),
}

_lib = None


def lib():
    """Load libnbbgpu.so (built in-tree).  Raises if it is missing -- no fallback."""
    global _lib
    if _lib is None:
        if not os.path.exists(SO_PATH):
            raise ImportError(f"{SO_PATH} is missing: build it with "
                              "`python -m paper_2110_12952_b200.build` (nvcc, sm_100a)")
        L = C.CDLL(SO_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(status: int) -> None:
    if status != 0:
        msg = lib().nbbgpu_last_error().decode(errors="replace")
        raise STATUS_TO_ERROR.get(status, NbbError)(msg)


def replica_array(replicas):
    flat = [int(v) for xy in replicas for v in xy]
    return (C.c_int32 * max(1, len(flat)))(*flat)
