"""Drop-in replacement of the reference engine's public entry points.

Same names, arguments, return types and error classes as
``ruleblock.engine`` (pkg/src/ruleblock/engine.py:41-62, 287-335, 342-368,
619-681); the evaluation itself runs in librbgpu.so on one sm_100a GPU.

What maps to what:

* ``EngineConfig`` -- same fields and validation (engine.py:41-62).
  ``symmetric_mode`` and ``enumerate_witnesses`` change results; the
  scheduling knobs (n_t, n_w, lanes_per_block, num_blocks, stealing,
  buffer_half_capacity, chunk_size) never changed results in the reference
  (engine.py:323-333 test) and are accepted for compatibility: on the GPU the
  schedule is persistent CTAs pulling (row block x column chunk) items from
  an atomic counter.
* ``PathProgram`` -- the path compiled against one encoding, here also
  resident on the device (instructions, slot descriptors, exact tables).
* ``run_partition`` / ``run_cross`` -- one kernel launch each; results are
  deduplicated like ``_dedup_witnesses`` (engine.py:600-616).
"""

from __future__ import annotations

import os
import threading
import time
import weakref
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from ._lib import RB_ENUMERATE, RB_EXACT_STATS, RB_STATS, RB_SYMMETRIC, check, i32, lib, ptr
from .encode import COL_CHARS, COL_CODES, COL_MASK, COL_TOKENS, Encoded, RelationEncoding, compile_program
from .errors import ConfigError, SchemaError

STEALING_MODES = ("off", "inter", "inter+intra")


@dataclass
class EngineConfig:
    n_t: int = 256
    n_w: int = 1024
    lanes_per_block: int = 32
    num_blocks: Optional[int] = None
    symmetric_mode: bool = True
    stealing: str = "inter+intra"
    buffer_half_capacity: int = 4096
    chunk_size: int = 4096
    enumerate_witnesses: bool = False
    device_stats: bool = True  # per-slot exact-evaluation counters (RB_STATS)
    # slot_evals = first-touch evaluations over EVERY pair (evaluate_pair,
    # engine.py:122-128; SURVEY 8d's E_s) from an extra exact pass
    # (RB_EXACT_STATS); off: the counts of the pairs the filter passed on
    exact_slot_evals: bool = False

    def __post_init__(self) -> None:
        if self.n_t < 1 or self.n_w < 1 or self.lanes_per_block < 1:
            raise ConfigError("n_t, n_w and lanes_per_block must all be >= 1")
        if self.stealing not in STEALING_MODES:
            raise ConfigError(f"stealing must be one of {STEALING_MODES}, got {self.stealing!r}")
        if self.buffer_half_capacity < 1 or self.chunk_size < 1:
            raise ConfigError("buffer_half_capacity and chunk_size must be >= 1")

    @classmethod
    def of(cls, cfg) -> "EngineConfig":
        """This package's EngineConfig for ``cfg``: None -> defaults, ours as
        is, any object with the reference's EngineConfig fields (engine.py:41-62,
        e.g. the reference's own, passed by its pipeline or CLI) converted
        field by field -- so the reference's call sites work unchanged."""
        if cfg is None:
            return cls()
        if isinstance(cfg, cls):
            return cfg
        names = [f for f in cls.__dataclass_fields__ if f not in ("device_stats", "exact_slot_evals")]
        return cls(**{f: getattr(cfg, f) for f in names if hasattr(cfg, f)})

    def resolved_blocks(self) -> int:
        return self.num_blocks if self.num_blocks else (os.cpu_count() or 1)

    def flags(self) -> int:
        f = RB_SYMMETRIC if self.symmetric_mode else 0
        if self.enumerate_witnesses:
            f |= RB_ENUMERATE
        if self.device_stats:
            f |= RB_STATS
        if self.exact_slot_evals:
            f |= RB_EXACT_STATS
        return f


@dataclass
class BlockStats:
    block_id: int
    intervals_processed: int = 0
    intervals_stolen: int = 0
    range_steals: int = 0
    comparisons: int = 0
    index_jumps: int = 0
    busy_s: float = 0.0
    slot_evals: Optional[np.ndarray] = None
    emitted: int = 0
    survivors: int = 0  # pairs the phase-1 filter could not rule out


@dataclass
class RunStats:
    blocks: list = field(default_factory=list)
    wall_s: float = 0.0
    n_intervals: int = 0
    kernel_ms: float = 0.0
    launches: int = 0
    specialized: bool = False  # the NVRTC-specialised pair kernel ran
    jit_log: str = ""

    def total_comparisons(self) -> int:
        return sum(b.comparisons for b in self.blocks)

    def describe(self) -> str:
        lines = [f"wall_s={self.wall_s:.4f} intervals={self.n_intervals} kernel_ms={self.kernel_ms:.3f}"]
        for b in self.blocks:
            lines.append(
                f"block {b.block_id}: comparisons={b.comparisons} survivors={b.survivors} emitted={b.emitted}"
            )
        return "\n".join(lines)


class CandidateSet:
    """Surviving pairs ``(t_tid, s_tid, rule_id)`` plus statistics.  The
    rows are held as arrays; ``pairs`` materialises the reference's list of
    tuples on first use."""

    def __init__(self, pairs=None, stats: Optional[RunStats] = None, *, arrays=None, rule_ids=None):
        self.stats = stats if stats is not None else RunStats()
        self._pairs = list(pairs) if pairs is not None else None
        self._arrays = arrays  # (t, s, rule_index) integer arrays of k rows (int64, or int32 as copied back)
        self._rule_ids = list(rule_ids) if rule_ids is not None else []

    @property
    def pairs(self) -> list:
        if self._pairs is None:
            t, s, r = self._arrays
            ids = self._rule_ids
            self._pairs = [(a, b, ids[k]) for a, b, k in zip(t.tolist(), s.tolist(), r.tolist())]
        return self._pairs

    @property
    def arrays(self):
        """(t, s, rule_index) integer arrays."""
        if self._arrays is None:
            idx = {rid: k for k, rid in enumerate(self._rule_ids)}
            p = self._pairs or []
            self._arrays = (
                np.array([x[0] for x in p], dtype=np.int64),
                np.array([x[1] for x in p], dtype=np.int64),
                np.array([idx.get(x[2], -1) for x in p], dtype=np.int64),
            )
        return self._arrays

    def pair_set(self) -> set:
        t, s, _ = self.arrays
        return set(zip(t.tolist(), s.tolist()))

    def sorted_pairs(self) -> list:
        return sorted(self.pairs)

    def __len__(self) -> int:
        return len(self._pairs) if self._pairs is not None else len(self._arrays[0])


# ---------------------------------------------------------------------------
# device objects


def default_device() -> int:
    return int(os.environ.get("RB_DEVICE", os.environ.get("LOCAL_RANK", "0")))


class Context:
    """One rb_ctx (device + stream).  One per (host thread, device)."""

    def __init__(self, device: int):
        h = _lib.c_vp()
        check(lib().rb_ctx_create(int(device), _lib.ctypes.byref(h)))
        self.handle = h
        self.device = int(device)
        self._fin = weakref.finalize(self, lib().rb_ctx_destroy, h)

    def set_stream(self, cuda_stream: int) -> None:
        check(lib().rb_ctx_set_stream(self.handle, _lib.c_vp(cuda_stream)))


_tls = threading.local()


def context(device: Optional[int] = None) -> Context:
    device = default_device() if device is None else int(device)
    cache = getattr(_tls, "ctx", None)
    if cache is None:
        cache = _tls.ctx = {}
    if device not in cache:
        cache[device] = Context(device)
    return cache[device]


class DeviceRelation:
    """An ``Encoded`` uploaded to one device (rb_rel).  Columns added to
    the encoding later are appended on the next ``sync``."""

    def __init__(self, ctx: Context, enc: Encoded):
        h = _lib.c_vp()
        check(lib().rb_relation_create(ctx.handle, enc.n, _lib.ctypes.byref(h)))
        self.handle = h
        self.ctx = ctx
        self.enc = enc
        self.n_uploaded = 0
        self._fin = weakref.finalize(self, lib().rb_relation_destroy, h)
        self.sync()

    def close(self) -> None:
        self._fin()

    def sync(self) -> None:
        L = lib()
        while self.n_uploaded < len(self.enc.columns):
            c = self.enc.columns[self.n_uploaded]
            col = _lib.ctypes.c_int32(-1)
            if c.kind == COL_CODES:
                data = i32(c.data)
                check(L.rb_relation_add_codes(self.handle, ptr(data), _lib.ctypes.byref(col)))
            elif c.kind == COL_MASK:
                data = np.ascontiguousarray(c.data, dtype=np.uint8)
                check(L.rb_relation_add_mask(self.handle, ptr(data), _lib.ctypes.byref(col)))
            elif c.kind == COL_TOKENS:
                offs = np.ascontiguousarray(c.offsets, dtype=np.int64)
                ids = i32(c.data)
                miss = None if c.missing is None else np.ascontiguousarray(c.missing, dtype=np.uint8)
                check(L.rb_relation_add_tokens(self.handle, ptr(offs), ptr(ids), ptr(miss), _lib.ctypes.byref(col)))
            elif c.kind == COL_CHARS:
                offs = np.ascontiguousarray(c.offsets, dtype=np.int64)
                data = np.ascontiguousarray(c.data)
                miss = None if c.missing is None else np.ascontiguousarray(c.missing, dtype=np.uint8)
                check(
                    L.rb_relation_add_chars(
                        self.handle, ptr(offs), ptr(data), c.width, ptr(miss), _lib.ctypes.byref(col)
                    )
                )
            else:
                raise ConfigError(f"unknown column kind {c.kind}")
            if col.value != self.n_uploaded:
                raise ConfigError("device column order diverged from the encoding")
            self.n_uploaded += 1


_dev_rel_cache: dict = {}


def device_relation(ctx: Context, enc: Encoded) -> DeviceRelation:
    key = (id(ctx), id(enc))
    dr = _dev_rel_cache.get(key)
    if dr is None or dr.enc is not enc or dr.ctx is not ctx:
        dr = DeviceRelation(ctx, enc)
        _dev_rel_cache[key] = dr
        weakref.finalize(enc, _dev_rel_cache.pop, key, None)
    dr.sync()
    return dr


class PathProgram:
    """A path compiled against one encoding and resident on one device
    (the reference's PathProgram, engine.py:342-368)."""

    def __init__(self, path, enc: Encoded, reg=None, device: Optional[int] = None, *, compiled=None,
                 drel: Optional[DeviceRelation] = None, ctx: Optional[Context] = None):
        self.path = path
        self.enc = enc
        self.n_slots = len(path.predicate_table)
        self.program = compiled if compiled is not None else compile_program(path, enc, reg)
        self.rule_ids = list(path.rule_ids)
        # ctx: the context (stream) the program runs on; a relation uploaded
        # through another context of the same device is shared, not copied
        self.ctx = ctx if ctx is not None else (context(device) if drel is None else drel.ctx)
        self.drel = drel if drel is not None else device_relation(self.ctx, enc)
        h = _lib.c_vp()
        p = self.program
        check(
            lib().rb_program_create(
                self.ctx.handle, self.drel.handle,
                ptr(p.ins_op), ptr(p.ins_slot), ptr(p.ins_fail), ptr(p.ins_rule), len(p.ins_op),
                ptr(p.slots), p.n_slots, ptr(p.tables), len(p.tables), _lib.ctypes.byref(h),
            )
        )
        self.handle = h
        self._fin = weakref.finalize(self, lib().rb_program_destroy, h)
        spec = _lib.ctypes.c_int32(0)
        cms = _lib.ctypes.c_double(0)
        log = _lib.ctypes.c_char_p()
        check(lib().rb_program_kernel_info(h, _lib.ctypes.byref(spec), _lib.ctypes.byref(cms), _lib.ctypes.byref(log)))
        self.specialized = bool(spec.value)
        self.jit_compile_ms = float(cms.value)
        self.jit_log = (log.value or b"").decode(errors="replace")

    def close(self) -> None:
        self._fin()

    # -- device-resident results -----------------------------------------

    def run_parts(self, parts, flags: int, rank: int = 0, world: int = 1) -> "DeviceResult":
        """Every partition with pairs and every pull of a device partition
        set (``pipeline.DeviceParts``) that rank ``rank`` of ``world`` owns,
        in one batched run (rb_run_parts).  The rows stay on the device."""
        res = _lib.c_vp()
        check(lib().rb_run_parts(self.ctx.handle, self.drel.handle, self.handle, parts.handle, int(rank), int(world),
                                 int(flags), _lib.ctypes.byref(res)))
        return DeviceResult(res, self.ctx)

    # -- raw runs ---------------------------------------------------------

    def run_batch(self, refs, offsets, splits, flags: int, out=None, implied: int = 0):
        """One launch over many partitions / cross blocks laid out back to
        back (rb_run_batch).  Returns ((t, s, rule, part) int32 arrays, rb_stats).
        ``out``: optional (t, s, rule, part) int32 host arrays the rows are
        copied into when they fit (see run_raw).  ``implied``: a bit mask of
        path slots every pair of every part holds (rb_run_batch_implied)."""
        L = lib()
        res = _lib.c_vp()
        refs_a = i32(refs)
        offs = np.ascontiguousarray(offsets, dtype=np.int64)
        spl = None if splits is None else np.ascontiguousarray(splits, dtype=np.int64)
        check(L.rb_run_batch_implied(self.ctx.handle, self.drel.handle, self.handle, ptr(refs_a), ptr(offs), ptr(spl),
                                     len(offs) - 1, flags, int(implied), _lib.ctypes.byref(res)))
        try:
            cnt = _lib.ctypes.c_int64(0)
            check(L.rb_result_count(res, _lib.ctypes.byref(cnt)))
            k = cnt.value
            if out is not None and all(len(a) >= k and a.dtype == np.int32 and a.flags["C_CONTIGUOUS"] for a in out):
                t, s, r, p = (a[:k] for a in out)
            else:
                t, s, r, p = (np.empty(k, dtype=np.int32) for _ in range(4))
            if k:
                check(L.rb_result_copy(res, ptr(t), ptr(s), ptr(r)))
                check(L.rb_result_copy_parts(res, ptr(p)))
            st = _lib.RbStats()
            check(L.rb_result_stats(res, _lib.ctypes.byref(st)))
        finally:
            L.rb_result_destroy(res)
        return (t, s, r, p), st

    def run_raw(self, refs, n: int, flags: int, *, split: int = -1, row_lo: int = 0, row_hi: Optional[int] = None,
                out=None):
        """Evaluate on the device.  Returns ((t, s, rule) int32 arrays, rb_stats).
        ``out``: optional (t, s, rule) int32 host arrays (e.g. pinned) the rows
        are copied into when they fit; the returned arrays are then views."""
        L = lib()
        res = _lib.c_vp()
        refs_a = None if refs is None else i32(refs)
        if split >= 0:
            left, right = refs_a[:split], refs_a[split:]
            check(L.rb_run_cross(self.ctx.handle, self.drel.handle, self.handle, ptr(np.ascontiguousarray(left)),
                                 len(left), ptr(np.ascontiguousarray(right)), len(right), flags,
                                 _lib.ctypes.byref(res)))
        elif row_lo <= 0 and (row_hi is None or row_hi >= n):
            check(L.rb_run_partition(self.ctx.handle, self.drel.handle, self.handle, ptr(refs_a), n, flags,
                                     _lib.ctypes.byref(res)))
        else:
            check(L.rb_run_partition_rows(self.ctx.handle, self.drel.handle, self.handle, ptr(refs_a), n,
                                          row_lo, n if row_hi is None else row_hi, flags, _lib.ctypes.byref(res)))
        try:
            cnt = _lib.ctypes.c_int64(0)
            check(L.rb_result_count(res, _lib.ctypes.byref(cnt)))
            k = cnt.value
            if out is not None and all(len(a) >= k and a.dtype == np.int32 and a.flags["C_CONTIGUOUS"] for a in out):
                t, s, r = (a[:k] for a in out)
            else:
                t = np.empty(k, dtype=np.int32)
                s = np.empty(k, dtype=np.int32)
                r = np.empty(k, dtype=np.int32)
            if k:
                check(L.rb_result_copy(res, ptr(t), ptr(s), ptr(r)))
            st = _lib.RbStats()
            check(L.rb_result_stats(res, _lib.ctypes.byref(st)))
        finally:
            L.rb_result_destroy(res)
        return (t, s, r), st


class DeviceResult:
    """An rb_result kept on the device: rows (t, s, rule) in HBM until copied.
    ``collect`` deduplicates them in place (rb_result_collect)."""

    def __init__(self, handle, ctx: Context):
        self.handle = handle
        self.ctx = ctx
        self._fin = weakref.finalize(self, lib().rb_result_destroy, handle)

    def close(self) -> None:
        self._fin()

    @property
    def count(self) -> int:
        cnt = _lib.ctypes.c_int64(0)
        check(lib().rb_result_count(self.handle, _lib.ctypes.byref(cnt)))
        return cnt.value

    def stats(self):
        st = _lib.RbStats()
        check(lib().rb_result_stats(self.handle, _lib.ctypes.byref(st)))
        return st

    def collect(self, n_tuples: int, n_rules: int) -> "DeviceResult":
        """pipeline.py:407-421 on the device: rows sorted by (t, s), the
        smallest rule index per (t, s)."""
        check(lib().rb_result_collect(self.handle, int(n_tuples), int(n_rules)))
        return self

    def copy(self, out=None):
        """(t, s, rule) int32 host arrays (into ``out`` when it fits)."""
        k = self.count
        if out is not None and all(len(a) >= k and a.dtype == np.int32 and a.flags["C_CONTIGUOUS"] for a in out):
            t, s, r = (a[:k] for a in out)
        else:
            t, s, r = (np.empty(k, dtype=np.int32) for _ in range(3))
        if k:
            check(lib().rb_result_copy(self.handle, ptr(t), ptr(s), ptr(r)))
        return t, s, r

    def torch_rows(self):
        """(t, s, rule) int32 torch tensors on the result's device: copies
        that stay valid after close().  The copies run on torch's current
        stream and are complete on return, so the library may free or reuse
        its buffers (rb_result_destroy, next run) right after."""
        import torch

        dev = torch.device("cuda", self.ctx.device)
        k = self.count
        out = [torch.empty(k, dtype=torch.int32, device=dev) for _ in range(3)]
        if k:
            from .distributed import _DevRows

            for o, p in zip(out, self.device_pointers()):  # the rows are final: rb_* returned after a sync
                o.copy_(torch.as_tensor(_DevRows(p, k), device=dev))
            torch.cuda.current_stream(dev).synchronize()
        return tuple(out)

    def torch_views(self):
        """(t, s, rule) int32 torch tensors viewing the result's device
        buffers (no copy): valid until close()."""
        import torch

        from .distributed import _DevRows

        dev = torch.device("cuda", self.ctx.device)
        k = self.count
        if k == 0:
            return tuple(torch.empty(0, dtype=torch.int32, device=dev) for _ in range(3))
        return tuple(torch.as_tensor(_DevRows(p, k), device=dev) for p in self.device_pointers())

    def device_pointers(self):
        """(t, s, rule) device addresses, valid until close()."""
        pt, ps, pr = _lib.c_vp(), _lib.c_vp(), _lib.c_vp()
        check(lib().rb_result_device(self.handle, _lib.ctypes.byref(pt), _lib.ctypes.byref(ps),
                                     _lib.ctypes.byref(pr), None))
        return pt.value, ps.value, pr.value


# ---------------------------------------------------------------------------
# reference-facing API


@dataclass
class PairBitmaps:
    """Per-pair reuse / value bits and evaluation counts (engine.py:69-90)."""

    reuse: np.ndarray
    value: np.ndarray
    scorer_calls: np.ndarray

    @classmethod
    def for_path(cls, path) -> "PairBitmaps":
        n = len(path.predicate_table)
        return cls(np.zeros(n, dtype=bool), np.zeros(n, dtype=bool), np.zeros(n, dtype=np.int64))

    def reset(self) -> None:
        self.reuse[:] = False
        self.value[:] = False
        self.scorer_calls[:] = 0


def evaluate_pair(path, t, s, bitmaps: PairBitmaps, reg=None, schema=None, all_witnesses: bool = False):
    """The sequential per-pair interpreter (engine.py:93-132), evaluated on
    the device: a two-tuple relation (t, s) run as one ordered cross pair.
    Returns the first witness rule id (or None), or every witness when
    ``all_witnesses``.  ``bitmaps.scorer_calls`` receives the first-touch
    evaluations per slot of the pair (RB_EXACT_STATS: the reference's own
    counts).  One call is one small launch; ``evaluate_pairs`` decides many
    pairs of a relation in one."""
    from .relation import Relation as _Relation
    from .relation import Schema as _Schema
    from .relation import TupleRecord as _TR

    if schema is None:
        raise ConfigError("evaluate_pair needs the relation schema")
    sch = _Schema(attributes=tuple((n, k) for n, k in schema.attributes))
    rel = _Relation(schema=sch, tuples=(_TR(0, t.eid, tuple(t.values)), _TR(1, s.eid, tuple(s.values))))
    enc = RelationEncoding(rel).prepare(list(path.predicate_table))
    prog = PathProgram(path, enc, reg)
    flags = RB_STATS | RB_EXACT_STATS | (RB_ENUMERATE if all_witnesses else 0)
    (tt, ss, rr), st = prog.run_raw(np.array([0, 1], dtype=np.int32), 2, flags, split=1)
    bitmaps.scorer_calls += np.array(st.slot_evals[: prog.n_slots], dtype=np.int64)
    bitmaps.reuse |= bitmaps.scorer_calls > 0
    order = {rid: k for k, rid in enumerate(path.checkpoint_order())}
    hits = sorted((prog.rule_ids[k] for k in rr.tolist()), key=lambda rid: order[rid])
    if all_witnesses:
        return hits
    return hits[0] if hits else None


def evaluate_pairs(path, relation, pairs, reg=None, encoded=None, program=None, all_witnesses: bool = False) -> list:
    """evaluate_pair for many (t_tid, s_tid) pairs of one relation in one
    device launch (each pair an ordered 1 x 1 cross block: t is the left
    tuple).  Returns, per pair, the first witness rule id (or None), or the
    list of every witness in path order when ``all_witnesses``."""
    prog = _program_for(path, relation, reg, encoded, program)
    pairs = np.asarray(pairs, dtype=np.int32).reshape(-1, 2)
    k = len(pairs)
    if k == 0:
        return []
    refs = np.ascontiguousarray(pairs.reshape(-1))
    offs = np.arange(0, 2 * k + 1, 2, dtype=np.int64)
    flags = RB_ENUMERATE if all_witnesses else 0
    (tt, ss, rr, pp), _ = prog.run_batch(refs, offs, np.ones(k, dtype=np.int64), flags)
    order = {rid: j for j, rid in enumerate(path.checkpoint_order())}
    hits: list = [[] for _ in range(k)]
    for p, r in zip(pp.tolist(), rr.tolist()):
        hits[p].append(prog.rule_ids[r])
    out = []
    for h in hits:
        h.sort(key=lambda rid: order[rid])
        out.append(h if all_witnesses else (h[0] if h else None))
    return out


def _dedup(t, s, r, symmetric: bool, enumerate_all: bool):
    """engine.py:600-616 on arrays: enumerate -> unique rows; symmetric ->
    the smallest rule index per (t, s); asymmetric -> rows as they are."""
    t = t.astype(np.int64)
    s = s.astype(np.int64)
    r = r.astype(np.int64)
    if len(t) == 0 or (not enumerate_all and not symmetric):
        return t, s, r
    order = np.lexsort((r, s, t))
    t, s, r = t[order], s[order], r[order]
    if enumerate_all:
        keep = np.ones(len(t), dtype=bool)
        keep[1:] = (t[1:] != t[:-1]) | (s[1:] != s[:-1]) | (r[1:] != r[:-1])
    else:
        keep = np.ones(len(t), dtype=bool)
        keep[1:] = (t[1:] != t[:-1]) | (s[1:] != s[:-1])
    return t[keep], s[keep], r[keep]


_enc_cache: dict = {}


def _encoding_for(relation, encoded):
    if isinstance(encoded, Encoded):
        return encoded
    key = id(relation)
    hit = _enc_cache.get(key)
    if hit is not None and hit.relation is relation:
        return hit
    enc = RelationEncoding(relation)
    _enc_cache[key] = enc
    try:
        weakref.finalize(relation, _enc_cache.pop, key, None)
    except TypeError:
        pass
    return enc


def _program_for(path, relation, reg, encoded, program) -> PathProgram:
    if isinstance(program, PathProgram):
        return program
    enc = _encoding_for(relation, encoded)
    if isinstance(enc, RelationEncoding):
        enc.prepare(list(path.predicate_table))
    return PathProgram(path, enc, reg)


def _refs_array(partition) -> np.ndarray:
    refs = np.asarray(partition.tuple_refs, dtype=np.int64)
    if len(np.unique(refs)) != len(refs):
        raise SchemaError(f"partition {getattr(partition, 'pid', '?')} has duplicate tuple refs")
    return refs.astype(np.int32)


def _candidates(prog: PathProgram, rows, st, cfg: EngineConfig, n_outer: int, wall: float) -> CandidateSet:
    # One partition (or one cross run over disjoint sides) evaluates every
    # pair once and reaches every checkpoint at most once per pair, so the
    # rows are already what _dedup_witnesses (engine.py:600-616) returns.
    t, s, r = (a.astype(np.int64) for a in rows)
    block = BlockStats(
        block_id=0,
        intervals_processed=max(1, -(-n_outer // cfg.n_t)),
        comparisons=int(st.comparisons),
        busy_s=st.kernel_ms / 1e3,
        slot_evals=np.array(st.slot_evals[: prog.n_slots], dtype=np.int64),
        emitted=int(st.emitted),
        survivors=int(st.survivors),
    )
    stats = RunStats(
        blocks=[block],
        wall_s=wall,
        n_intervals=max(1, -(-n_outer // cfg.n_t)),
        kernel_ms=float(st.kernel_ms),
        launches=int(st.launches),
        specialized=bool(st.specialized),
        jit_log=prog.jit_log,
    )
    return CandidateSet(stats=stats, arrays=(t, s, r), rule_ids=prog.rule_ids)


def run_partition(partition, relation, path, cfg=None, reg=None, encoded=None, program=None) -> CandidateSet:
    """All pairs of one partition (engine.py:619-646): symmetric i<j with
    t = the lower position, or every ordered i != j."""
    cfg = EngineConfig.of(cfg)
    if partition is None or len(partition.tuple_refs) == 0:
        return CandidateSet(pairs=[])
    started = time.perf_counter()
    prog = _program_for(path, relation, reg, encoded, program)
    refs = _refs_array(partition)
    rows, st = prog.run_raw(refs, len(refs), cfg.flags())
    return _candidates(prog, rows, st, cfg, len(refs), time.perf_counter() - started)


def split_rows_by_pairs(n: int, parts: int, symmetric: bool = True) -> list[tuple[int, int]]:
    """Cut outer positions [0, n) into `parts` contiguous ranges of (nearly)
    equal pair counts -- row i owns n-1-i pairs in symmetric mode, n-1
    otherwise.  The unit of multi-GPU sharding of one partition."""
    if parts < 1:
        raise ConfigError("parts must be >= 1")
    if not symmetric:
        cuts = [round(k * n / parts) for k in range(parts + 1)]
    else:
        total = n * (n - 1) // 2

        def before(r: int) -> int:  # pairs owned by rows < r
            return r * n - r * (r + 1) // 2

        cuts = [0]
        for k in range(1, parts):
            goal = total * k // parts
            lo, hi = cuts[-1], n
            while lo < hi:
                mid = (lo + hi) // 2
                if before(mid) < goal:
                    lo = mid + 1
                else:
                    hi = mid
            cuts.append(lo)
        cuts.append(n)
    return [(cuts[k], cuts[k + 1]) for k in range(parts)]


def run_partition_rows(partition, relation, path, row_lo: int, row_hi: int, cfg=None, reg=None, encoded=None,
                       program=None) -> CandidateSet:
    """The pairs of `partition` whose outer (t) position lies in [row_lo,
    row_hi): one shard of run_partition.  The union over a split of [0, n)
    equals run_partition exactly."""
    cfg = EngineConfig.of(cfg)
    if partition is None or len(partition.tuple_refs) == 0:
        return CandidateSet(pairs=[])
    started = time.perf_counter()
    prog = _program_for(path, relation, reg, encoded, program)
    refs = _refs_array(partition)
    rows, st = prog.run_raw(refs, len(refs), cfg.flags(), row_lo=row_lo, row_hi=row_hi)
    return _candidates(prog, rows, st, cfg, max(0, row_hi - row_lo), time.perf_counter() - started)


def implied_slots_of(path, partitions) -> int:
    """The path slots every pair of these partitions holds: the equality root
    of the branch they were keyed on (DataPartition.branch_id, partitioning.py:
    93-131), when they all share it and none is the missing-value group
    (their key_group is known and is not the missing key).  0 otherwise."""
    bids = {getattr(p, "branch_id", None) for p in partitions}
    if len(bids) != 1:
        return 0
    b = bids.pop()
    roots = list(getattr(path, "root_slots", ()))
    if not isinstance(b, int) or not 0 <= b < len(roots):
        return 0
    s = roots[b]
    pred = path.predicate_table[s]
    if pred.comparator != "eq" or pred.is_cross_attr or pred.rhs_attr is None:
        return 0
    if any(getattr(p, "key_group", None) in (None, "\x00missing") for p in partitions):
        return 0
    return 1 << int(s)


def _batch(prog: PathProgram, blocks, cfg: EngineConfig, implied: int = 0):
    """blocks: list of (refs int32 array, split or -1).  One launch; returns
    one CandidateSet per block."""
    started = time.perf_counter()
    sizes = [len(r) for r, _ in blocks]
    offsets = np.zeros(len(blocks) + 1, dtype=np.int64)
    np.cumsum(sizes, out=offsets[1:])
    refs = np.concatenate([r for r, _ in blocks]) if blocks else np.zeros(0, np.int32)
    splits = np.array([sp for _, sp in blocks], dtype=np.int64)
    (t, s, r, p), st = prog.run_batch(refs, offsets, splits, cfg.flags(), implied=implied)
    wall = time.perf_counter() - started
    order = np.argsort(p, kind="stable")
    t, s, r, p = t[order], s[order], r[order], p[order]
    bounds = np.searchsorted(p, np.arange(len(blocks) + 1))
    out = []
    for k, (refs_k, sp) in enumerate(blocks):
        a, b = bounds[k], bounds[k + 1]
        n = len(refs_k)
        if sp >= 0:
            cmp = sp * (n - sp)
        elif cfg.symmetric_mode:
            cmp = n * (n - 1) // 2
        else:
            cmp = n * (n - 1)
        tt, ss, rr = (x[a:b].astype(np.int64) for x in (t, s, r))  # unique per block by construction
        block = BlockStats(block_id=0, intervals_processed=1, comparisons=int(cmp), emitted=int(b - a),
                           slot_evals=np.zeros(prog.n_slots, dtype=np.int64))
        stats = RunStats(blocks=[block], wall_s=wall, n_intervals=1, kernel_ms=float(st.kernel_ms),
                         launches=int(st.launches), specialized=bool(st.specialized), jit_log=prog.jit_log)
        out.append(CandidateSet(stats=stats, arrays=(tt, ss, rr), rule_ids=prog.rule_ids))
    if sum(b.stats.total_comparisons() for b in out) != int(st.comparisons):
        raise ConfigError("device pair count disagrees with the batch layout")
    return out


SPLIT_PAIRS = 10_000_000_000  # a mixed-branch batch this large splits off its dominant branch (one extra launch)


def split_by_root(masks, pairs):
    """Batches of unit indices for a batch mixing branches: the dominant
    implied root (at least half the pairs, when the batch has SPLIT_PAIRS
    pairs or more) in a batch of its own, regated; the rest in one batch with
    the roots common to all of it.  Returns [(indices, implied mask)]."""
    total = sum(pairs)
    kinds = set(masks)
    if len(kinds) == 1:
        return [(list(range(len(masks))), masks[0] if masks else 0)]
    by = {}
    for m, c in zip(masks, pairs):
        by[m] = by.get(m, 0) + c
    dom = max(by, key=by.get)
    if total < SPLIT_PAIRS or dom == 0 or 2 * by[dom] < total:
        return [(list(range(len(masks))), 0)]
    rest = [k for k, m in enumerate(masks) if m != dom]
    rest_masks = {masks[k] for k in rest}
    return [([k for k, m in enumerate(masks) if m == dom], dom),
            (rest, rest_masks.pop() if len(rest_masks) == 1 else 0)]


def _batched(prog, path, units, blocks, cfg, symmetric_units: bool) -> list:
    """_batch over `blocks` (one per unit), split by split_by_root."""
    def pairs_of(b):
        r, sp = b
        return sp * (len(r) - sp) if sp >= 0 else len(r) * (len(r) - 1) // 2
    masks = [implied_slots_of(path, u) for u in units]
    groups = split_by_root(masks, [pairs_of(b) for b in blocks])
    if len(groups) == 1:
        return _batch(prog, blocks, cfg, groups[0][1])
    out = [None] * len(blocks)
    for idx, m in groups:
        for k, cs in zip(idx, _batch(prog, [blocks[k] for k in idx], cfg, m)):
            out[k] = cs
    return out


def run_partitions(partitions, relation, path, cfg=None, reg=None, encoded=None, program=None) -> list:
    """run_partition over many partitions in ONE device launch (the
    pipeline's per-task loop, pipeline.py:177-209, batched) -- or one per
    branch when a large batch mixes equality-rooted branches (each runs with
    its root implied).  Returns one CandidateSet per partition, each
    identical to run_partition's."""
    cfg = EngineConfig.of(cfg)
    live = [p for p in partitions if p is not None and len(p.tuple_refs)]
    prog = _program_for(path, relation, reg, encoded, program)
    res = iter(_batched(prog, path, [[p] for p in live], [(_refs_array(p), -1) for p in live], cfg, True)) if live \
        else iter(())
    return [next(res) if (p is not None and len(p.tuple_refs)) else CandidateSet(pairs=[]) for p in partitions]


def run_crosses(pairs, relation, path, cfg=None, reg=None, encoded=None, program=None) -> list:
    """run_cross over many (left, right) partition pairs in one launch --
    e.g. the per-block record-linkage runs of BASELINE config 5."""
    cfg = EngineConfig.of(cfg)
    prog = _program_for(path, relation, reg, encoded, program)
    blocks = []
    for left, right in pairs:
        lr, rr = _refs_array(left), _refs_array(right)
        both = np.concatenate([lr, rr])
        if len(np.unique(both)) != len(both):
            raise SchemaError("partition -1 has duplicate tuple refs")
        blocks.append((both, len(lr)))
    return _batched(prog, path, [list(pr) for pr in pairs], blocks, cfg, False)


def run_cross(left, right, relation, path, cfg=None, reg=None, encoded=None, program=None) -> CandidateSet:
    """Every (t in left, s in right) pair, t always the left tuple
    (engine.py:649-681 with _bipartite_patch 684-719)."""
    cfg = EngineConfig.of(cfg)
    started = time.perf_counter()
    prog = _program_for(path, relation, reg, encoded, program)
    lrefs = _refs_array(left)
    rrefs = _refs_array(right)
    refs = np.concatenate([lrefs, rrefs])
    if len(np.unique(refs)) != len(refs):
        raise SchemaError("partition -1 has duplicate tuple refs")  # the combined partition (engine.py:671-675)
    rows, st = prog.run_raw(refs, len(refs), cfg.flags(), split=len(lrefs))
    return _candidates(prog, rows, st, cfg, len(lrefs), time.perf_counter() - started)
