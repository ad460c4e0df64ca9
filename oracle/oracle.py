"""ctypes wrapper of the CPU oracle (oracle/rb_oracle.c).

TEST INFRASTRUCTURE ONLY -- imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference leg, always as the checker or the
timed CPU baseline, never as the product path.  It restates the reference
engine's per-pair semantics (pkg/src/ruleblock/engine.py:93-132, 508-559;
encode.py:191-324; _kernels.py:29-83) in C; parity of this restatement is
pinned against the reference itself by tests/golden (see make_golden.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")


class OrcColumn(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32),
        ("width", ctypes.c_int32),
        ("data", ctypes.c_void_p),
        ("offsets", ctypes.c_void_p),
        ("missing", ctypes.c_void_p),
    ]


def build(force: bool = False) -> str:
    src = os.path.join(HERE, "rb_oracle.c")
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        L.orc_slot_size.restype = ctypes.c_int32
        L.orc_witness_pairs.restype = None
        L.orc_witness_pairs.argtypes = [
            ctypes.c_void_p,
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32,
            ctypes.c_void_p, ctypes.c_int32,
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p,
        ]
        L.orc_run.restype = ctypes.c_int64
        L.orc_run.argtypes = [
            ctypes.c_void_p, ctypes.c_int32,
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32,
            ctypes.c_void_p, ctypes.c_int32,
            ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
            ctypes.c_uint32, ctypes.c_int32,
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
            ctypes.POINTER(ctypes.c_int64), ctypes.c_void_p,
        ]
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data


def _columns(enc):
    keep = []
    cols = (OrcColumn * max(1, len(enc.columns)))()
    for k, c in enumerate(enc.columns):
        data = np.ascontiguousarray(c.data)
        offs = None if c.offsets is None else np.ascontiguousarray(c.offsets, dtype=np.int64)
        miss = None if c.missing is None else np.ascontiguousarray(c.missing, dtype=np.uint8)
        keep += [data, offs, miss]
        cols[k].kind = c.kind
        cols[k].width = c.width
        cols[k].data = _ptr(data)
        cols[k].offsets = _ptr(offs)
        cols[k].missing = _ptr(miss)
    return cols, keep


def witness(enc, prog, t, s, *, nthreads=0):
    """Rule of the first checkpoint each pair (t[k], s[k]) reaches, evaluated
    t-then-s (engine.py:531-559, first witness); -1 where no rule holds."""
    L = lib()
    cols, keep = _columns(enc)
    t = np.ascontiguousarray(t, dtype=np.int32)
    s = np.ascontiguousarray(s, dtype=np.int32)
    out = np.empty(len(t), dtype=np.int32)
    slots = np.ascontiguousarray(prog.slots)
    L.orc_witness_pairs(cols, _ptr(prog.ins_op), _ptr(prog.ins_slot), _ptr(prog.ins_fail), _ptr(prog.ins_rule),
                        len(prog.ins_op), _ptr(slots), prog.n_slots, _ptr(t), _ptr(s), len(t), nthreads, _ptr(out))
    del keep
    return out


def run(enc, prog, refs, n, *, split=-1, row_lo=0, row_hi=None, flags=1, nthreads=0):
    """Evaluate pairs with the oracle.  ``refs`` is an int32 array of tids or
    None (identity).  Returns (rows int64 (k,3) [t, s, rule_index],
    comparisons, slot_evals)."""
    L = lib()
    keep = []
    cols = (OrcColumn * max(1, len(enc.columns)))()
    for k, c in enumerate(enc.columns):
        data = np.ascontiguousarray(c.data)
        offs = None if c.offsets is None else np.ascontiguousarray(c.offsets, dtype=np.int64)
        miss = None if c.missing is None else np.ascontiguousarray(c.missing, dtype=np.uint8)
        keep += [data, offs, miss]
        cols[k].kind = c.kind
        cols[k].width = c.width
        cols[k].data = _ptr(data)
        cols[k].offsets = _ptr(offs)
        cols[k].missing = _ptr(miss)
    if refs is not None:
        refs = np.ascontiguousarray(refs, dtype=np.int32)
    row_hi = n if row_hi is None else row_hi
    slots = np.ascontiguousarray(prog.slots)
    cap = 1 << 16
    while True:
        t = np.empty(cap, dtype=np.int32)
        s = np.empty(cap, dtype=np.int32)
        r = np.empty(cap, dtype=np.int32)
        cmp = ctypes.c_int64(0)
        evals = np.zeros(64, dtype=np.int64)
        count = L.orc_run(
            cols, len(enc.columns),
            _ptr(prog.ins_op), _ptr(prog.ins_slot), _ptr(prog.ins_fail), _ptr(prog.ins_rule), len(prog.ins_op),
            _ptr(slots), prog.n_slots,
            _ptr(refs), n, split, row_lo, row_hi, flags, nthreads,
            _ptr(t), _ptr(s), _ptr(r), cap, ctypes.byref(cmp), _ptr(evals),
        )
        if count <= cap:
            rows = np.stack([t[:count], s[:count], r[:count]], axis=1).astype(np.int64)
            return rows, int(cmp.value), evals[: prog.n_slots].copy()
        cap = int(count)
