"""ctypes binding of librbgpu.so (include/rbgpu.h).

The shared library is built in-tree (``python -m paper_2410_04349_b200.build``
or ``__graft_entry__.build()``).  There is no fallback: if the library or a
usable sm_100 device is missing, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import re

import numpy as np

from .errors import ConfigError, RuleBlockError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "librbgpu.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "rbgpu.h")
HEADERS = [HEADER, os.path.join(os.path.dirname(HERE), "include", "rbencode.h")]

RB_OK = 0
RB_ERR_INVALID, RB_ERR_CUDA, RB_ERR_OOM, RB_ERR_LIMIT, RB_ERR_INTERNAL = -1, -2, -3, -4, -5
RB_SYMMETRIC, RB_ENUMERATE, RB_STATS, RB_EXACT_STATS = 1, 2, 4, 8
RB_PART_PULLS, RB_PART_KEYS_DEVICE = 1, 2
MAX_SLOTS = 64

c_i32p = ctypes.POINTER(ctypes.c_int32)
c_i64p = ctypes.POINTER(ctypes.c_int64)
c_vp = ctypes.c_void_p
c_vpp = ctypes.POINTER(ctypes.c_void_p)


class RbStats(ctypes.Structure):
    _fields_ = [
        ("comparisons", ctypes.c_int64),
        ("survivors", ctypes.c_int64),
        ("emitted", ctypes.c_int64),
        ("kernel_ms", ctypes.c_double),
        ("launches", ctypes.c_int32),
        ("retries", ctypes.c_int32),
        ("slot_evals", ctypes.c_int64 * MAX_SLOTS),
        ("specialized", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("jit_compile_ms", ctypes.c_double),
        ("pair_ms", ctypes.c_double),
    ]


_SIGNATURES = {
    "rb_last_error": (ctypes.c_char_p, []),
    "rb_version": (ctypes.c_char_p, []),
    "rb_ctx_create": (ctypes.c_int, [ctypes.c_int, c_vpp]),
    "rb_ctx_set_stream": (ctypes.c_int, [c_vp, c_vp]),
    "rb_ctx_destroy": (ctypes.c_int, [c_vp]),
    "rb_relation_create": (ctypes.c_int, [c_vp, ctypes.c_int64, c_vpp]),
    "rb_relation_add_codes": (ctypes.c_int, [c_vp, c_vp, c_i32p]),
    "rb_relation_add_mask": (ctypes.c_int, [c_vp, c_vp, c_i32p]),
    "rb_relation_add_tokens": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_i32p]),
    "rb_relation_add_chars": (ctypes.c_int, [c_vp, c_vp, c_vp, ctypes.c_int32, c_vp, c_i32p]),
    "rb_relation_destroy": (ctypes.c_int, [c_vp]),
    "rb_program_create": (
        ctypes.c_int,
        [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, ctypes.c_int32, c_vp, ctypes.c_int32, c_vp, ctypes.c_int64, c_vpp],
    ),
    "rb_program_destroy": (ctypes.c_int, [c_vp]),
    "rb_program_kernel_info": (
        ctypes.c_int, [c_vp, c_i32p, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_char_p)]),
    "rb_run_partition": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, ctypes.c_int64, ctypes.c_uint32, c_vpp]),
    "rb_run_partition_rows": (
        ctypes.c_int,
        [c_vp, c_vp, c_vp, c_vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_uint32, c_vpp],
    ),
    "rb_run_cross": (
        ctypes.c_int,
        [c_vp, c_vp, c_vp, c_vp, ctypes.c_int64, c_vp, ctypes.c_int64, ctypes.c_uint32, c_vpp],
    ),
    "rb_run_batch": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, ctypes.c_int32, ctypes.c_uint32, c_vpp]),
    "rb_run_batch_implied": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, ctypes.c_int32, ctypes.c_uint32,
                                            ctypes.c_uint64, c_vpp]),
    "rb_result_count": (ctypes.c_int, [c_vp, c_i64p]),
    "rb_result_copy_parts": (ctypes.c_int, [c_vp, c_vp]),
    "rb_result_copy": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp]),
    "rb_result_stats": (ctypes.c_int, [c_vp, ctypes.POINTER(RbStats)]),
    "rb_result_destroy": (ctypes.c_int, [c_vp]),
    "rb_result_device": (ctypes.c_int, [c_vp, c_vpp, c_vpp, c_vpp, c_vpp]),
    "rb_partition": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, c_vpp]),
    "rb_partition_codes": (
        ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, c_vpp]),
    "rb_parts_info": (ctypes.c_int, [c_vp, c_i64p, c_i64p, c_i64p, c_i64p]),
    "rb_parts_copy": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "rb_parts_destroy": (ctypes.c_int, [c_vp]),
    "rb_parts_set_roots": (ctypes.c_int, [c_vp, c_vp, c_vp, ctypes.c_int32]),
    "rb_run_parts": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_uint32, c_vpp]),
    "rb_result_collect": (ctypes.c_int, [c_vp, ctypes.c_int64, ctypes.c_int32]),
    "rb_collect_device": (
        ctypes.c_int,
        [c_vp, c_vp, c_vp, c_vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, c_vp, c_vp, c_vp, c_i64p]),
    # include/rbencode.h
    "rb_encode_eq_codes": (ctypes.c_int, [c_vp, c_vp, c_vp, ctypes.c_int64, c_vp]),
    "rb_encode_tokens": (ctypes.c_int64, [c_vp, c_vp, c_vp, ctypes.c_int64, c_vp, c_vp, c_i32p]),
    "rb_encode_chars": (ctypes.c_int64, [c_vp, c_vp, c_vp, ctypes.c_int64, c_vp, c_vp]),
    "rb_csv_parse": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_int64, c_vpp, c_i64p]),
    "rb_csv_shape": (ctypes.c_int, [c_vp, c_i64p, c_i32p]),
    "rb_csv_header": (ctypes.c_int, [c_vp, ctypes.c_int32, c_vpp, c_i64p]),
    "rb_csv_column": (ctypes.c_int, [c_vp, ctypes.c_int32, c_vpp, c_i64p, ctypes.POINTER(ctypes.POINTER(ctypes.c_int64))]),
    "rb_csv_free": (None, [c_vp]),
    "rb_parse_numbers": (None, [c_vp, c_vp, ctypes.c_int64, c_vp, c_vp]),
    "rb_token_counts": (None, [c_vp, c_vp, ctypes.c_int64, c_vp]),
}


def header_symbols() -> list[str]:
    """Every function the public headers declare."""
    out = []
    for h in HEADERS:
        out += re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\*?(rb_\w+)\s*\(", open(h).read(), flags=re.M)
    return out


_lib = None


def lib():
    """Load librbgpu.so (raises RuleBlockError when it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuleBlockError(
                f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                "(there is no CPU fallback for the rule-evaluation path)"
            )
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc == RB_OK:
        return
    msg = lib().rb_last_error().decode(errors="replace")
    if rc in (RB_ERR_INVALID, RB_ERR_LIMIT):
        raise ConfigError(msg)
    raise RuleBlockError(f"librbgpu error {rc}: {msg}")


def ptr(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def i32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int32)
