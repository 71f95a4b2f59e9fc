"""ctypes binding of libvqkv_b200.so (include/vqkv_c.h).

The library is the product's only compute path.  There is no CPU fallback:
if the shared library is missing or cannot be loaded, importing a compute
function raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

from .errors import raise_for_status

_PKG = os.path.dirname(os.path.abspath(__file__))
# VQKV_LIB: development override (A/B timing of two builds on one box)
LIB_PATH = os.environ.get("VQKV_LIB") or os.path.join(_PKG, "lib", "libvqkv_b200.so")

P = C.c_void_p
u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
fp = C.POINTER(C.c_float)


class AttendArgs(C.Structure):
    _fields_ = [
        ("n_pairs", C.c_uint32),
        ("group", C.c_uint32),
        ("q_dev", C.c_void_p),
        ("init_k_dev", C.c_void_p),
        ("init_v_dev", C.c_void_p),
        ("n_init", C.c_uint64),
        ("kcodes_dev", C.c_void_p),
        ("vcodes_dev", C.c_void_p),
        ("n_comp", C.c_uint64),
        ("local_k_dev", C.c_void_p),
        ("local_v_dev", C.c_void_p),
        ("n_local", C.c_uint64),
        ("scale", C.c_double),
        ("out_dev", C.c_void_p),
        ("lse_dev", C.c_void_p),
        ("init_stride", C.c_uint64),
        ("local_stride", C.c_uint64),
        ("kcodes_stride", C.c_uint64),
        ("vcodes_stride", C.c_uint64),
        ("kcodes_layout", C.c_uint32),
        ("kcodes_cap", C.c_uint64),
    ]


KEYCODES_ROWS, KEYCODES_GROUP_MAJOR = 0, 1


_SIGS = {
    "vqkv_last_error": (C.c_char_p, []),
    "vqkv_version": (C.c_char_p, []),
    "vqkv_launch_count": (C.c_uint64, []),
    "vqkv_set_encode_path": (C.c_int, [C.c_int]),
    "vqkv_stack_create": (C.c_int, [C.c_int, C.c_int, C.c_uint32, u32p, C.c_uint32, fp, fp, C.POINTER(P)]),
    "vqkv_stack_destroy": (C.c_int, [P]),
    "vqkv_stack_describe": (
        C.c_int,
        [P, u32p, u32p, u64p, C.POINTER(C.c_int), C.POINTER(C.c_int)],
    ),
    "vqkv_stack_stage_size": (C.c_int, [P, C.c_uint32, u32p]),
    "vqkv_stack_effective": (C.c_int, [P, C.c_uint32, fp, fp]),
    "vqkv_stack_effective_dev": (C.c_int, [P, C.c_uint32, C.POINTER(C.c_void_p)]),
    "vqkv_payload_bytes": (C.c_uint64, [P, C.c_uint64]),
    "vqkv_stack_take_error": (C.c_int, [P]),
    "vqkv_quantize_batch": (C.c_int, [P, P, C.c_uint32, C.c_uint64, C.c_uint64, P, P, P]),
    "vqkv_quantize_batch_ex": (C.c_int, [P, P, C.c_uint32, C.c_uint64, C.c_uint64, P, P, P, P]),
    "vqkv_quantize_batch_host": (C.c_int, [P, P, C.c_uint32, C.c_uint64, C.c_uint64, P, P, P]),
    "vqkv_quantize_batch_host_async": (C.c_int, [P, P, C.c_uint32, C.c_uint64, C.c_uint64, P, P, P]),
    "vqkv_nearest_batch": (C.c_int, [P, C.c_uint32, P, C.c_uint64, C.c_uint64, P, P, P]),
    "vqkv_reconstruct_block": (C.c_int, [P, P, C.c_uint32, C.c_uint64, C.c_uint64, C.c_uint64, P, P]),
    "vqkv_reconstruct_block_ex": (C.c_int, [P, P, C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64, C.c_uint64, P, P]),
    "vqkv_attend_decode": (C.c_int, [P, P, C.POINTER(AttendArgs), P]),
    "vqkv_lse_combine": (C.c_int, [P, P, C.c_uint32, C.c_uint64, C.c_uint32, P, P, P]),
    "vqkv_lse_allgather_combine": (C.c_int, [P, P, P, C.c_uint64, C.c_uint32, P, P, P, P, P]),
    "vqkv_nccl_comm_init_all": (C.c_int, [C.c_int, C.POINTER(C.c_int), C.POINTER(P)]),
    "vqkv_nccl_comm_destroy": (C.c_int, [P]),
    "vqkv_train_batch": (C.c_int, [P, P, C.c_uint64, C.c_float, C.c_float, C.c_int, P, C.POINTER(C.c_double), P]),
    "vqkv_train_batch_host": (C.c_int, [P, P, C.c_uint64, C.c_float, C.c_float, C.c_int, P, C.POINTER(C.c_double)]),
    "vqkv_encode_counters": (C.c_int, [P, u64p]),
    "vqkv_encode_phase_clocks": (C.c_int, [P, u64p]),
    "vqkv_payload_append": (C.c_int, [P, C.c_uint64, C.c_uint64, P, C.c_uint64, C.c_uint64, C.c_uint32, P]),
    "vqkv_keycodes_gm_bytes": (C.c_uint64, [P, C.c_uint64]),
    "vqkv_attend_gm_supported": (C.c_int, [P, P, C.POINTER(AttendArgs)]),
    "vqkv_keycodes_to_gm": (
        C.c_int,
        [P, P, C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64, P, C.c_uint64, C.c_uint64, C.c_uint64, P],
    ),
    "vqkv_keycodes_from_gm": (
        C.c_int,
        [P, P, C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint64, P, C.c_uint64, P],
    ),
    "vqkv_profile_enable": (C.c_int, [C.c_int]),
    "vqkv_profile_collect": (C.c_int, [C.c_char_p, C.POINTER(C.c_double), u64p]),
    "vqkv_generate_synthetic": (
        C.c_int,
        [C.c_int, C.c_uint32, C.c_uint64, C.c_uint32, C.c_uint64, C.c_double, C.c_float, C.c_float, P],
    ),
    "vqkv_random_stack": (C.c_int, [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, P, P]),
    "vqkv_fnv1a64": (C.c_uint64, [P, C.c_uint64]),
    "vqkv_quantize_rows_host": (C.c_int, [P, P, C.c_uint64, C.c_uint64, P, P, P]),
    "vqkv_nearest_host": (C.c_int, [P, C.c_uint32, P, C.c_uint64, u32p, fp]),
    "vqkv_reconstruct_block_host": (C.c_int, [P, P, C.c_uint64, C.c_uint64, C.c_uint64, P]),
    "vqkv_attend_decode_host": (C.c_int, [P, P, C.POINTER(AttendArgs)]),
    "vqkv_attend_raw_host": (C.c_int, [C.c_int, P, P, C.c_uint64, C.c_uint32, C.c_uint32, P, C.c_double, P]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def load():
    """Load (once) and return the ctypes handle; raise if it is absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"libvqkv_b200.so not found at {LIB_PATH}; build it with "
                "`python -m paper_2603_16435_b200.build` (no CPU fallback exists)"
            )
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def call(name, *args):
    """Call a status-returning entry point; raise the mirrored exception."""
    L = load()
    st = getattr(L, name)(*args)
    if st != 0:
        raise_for_status(st, L.vqkv_last_error().decode(errors="replace"))
    return st


def launch_count() -> int:
    return int(load().vqkv_launch_count())
