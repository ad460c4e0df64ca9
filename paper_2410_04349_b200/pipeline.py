"""The callers on either side of the path: plan-derived partitioning, the
device run over all partitions and pulls, and the collect step -- the
reference's pipeline_run (pkg/src/ruleblock/pipeline.py:245-433) with its
partitioning, execution and collect stages on the GPU.

Restates the reference's partitioning and pipeline:
  * one hash partitioner per root edge of the plan     partitioning.py:40-90
      eq edge  -> the canonical value ("n:<repr(float)>" / "v:<strip>")
      sim edge -> a minhash band over tokens (jaccard / exact_token) or
                  character 3-grams (edit), blake2b item hashes + splitmix
      cross-attribute edge -> one key group
  * groups in sorted-key order, oversize groups split round-robin into
    sibling sub-partitions                              partitioning.py:93-131
  * sibling pull pairs                                  partitioning.py:144-157
  * pipeline_run: single-partition threshold, skip single tuples, run every
    partition and pull, collect = union deduplicated per (t, s) keeping the
    earliest rule in rule-set order                     pipeline.py:245-433
The group keys are byte-identical to the reference's, so the partitions
(pids, refs, branches, sibling groups) are identical too.

Stages of ``pipeline_run``:
  * keys   (host): each root edge's key strings, ranked in sorted key-string
           order (one int64 per tuple and branch; minhash vectorised)
  * partition (GPU, rb_partition): stable radix sort of (key, tid) per
           branch, group sizes, round-robin sibling deal, pulls -- the sorted
           tuple ids stay in HBM as the refs of the run
  * execute (GPU, rb_run_parts): every partition with pairs and every pull
           in one batched run; several GPUs split the units by LPT
  * collect (GPU, rb_result_collect): radix sort of the rows on (t, s,
           rule), first row per (t, s)
Synthetic encoded relations (the benchmarks) key their equality roots on the
device code columns directly (``run_pipeline_encoded``): same groups, pids in
code order instead of key-string order, identical candidate set.
"""

from __future__ import annotations

import hashlib
import threading
import time
import weakref
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from .engine import CandidateSet, EngineConfig, RunStats
from .errors import ConfigError
from .plan import is_checkpoint
from .relation import DataPartition, is_missing, is_numeric_kind
from .text import fold_text, tokenize, value_text

MISSING_KEY = "\x00missing"
_MASK64 = (1 << 64) - 1


@dataclass
class BandingConfig:
    rows: int = 4  # minhash values concatenated into one band key (partitioning.py:34-37)
    seed: int = 0


@dataclass
class PipelineConfig:
    """pipeline.py:63-74.  ``async_mode`` / ``stage_queue_bound`` /
    ``rng_seed`` shaped the reference's host queues and CHBL placement and
    never changed results; they are accepted.  ``devices`` / ``workers_per_device``
    name the CUDA devices used when pipeline_run is not given any."""

    async_mode: bool = True
    stage_queue_bound: int = 8
    max_partition_size: int = 512
    enable_pulls: bool = False
    banding: BandingConfig = field(default_factory=BandingConfig)
    rng_seed: int = 0
    single_partition_threshold: Optional[int] = None  # None: follows max_partition_size
    devices: tuple = (0,)
    workers_per_device: int = 1


def stable_hash64(text: str, seed: int = 0) -> int:
    """hashing.py:17-19: blake2b-64 of the utf-8 bytes, salted with the seed."""
    d = hashlib.blake2b(text.encode("utf-8"), digest_size=8, salt=seed.to_bytes(8, "little", signed=False)).digest()
    return int.from_bytes(d, "little")


def mix64(values: np.ndarray, seed: int) -> np.ndarray:
    """hashing.py:27-37, the splitmix64-style mixer (uint64 wrap-around)."""
    x = values.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        x += np.uint64((seed * 0x9E3779B97F4A7C15) & _MASK64)
        x ^= x >> np.uint64(30)
        x *= np.uint64(0xBF58476D1CE4E5B9)
        x ^= x >> np.uint64(27)
        x *= np.uint64(0x94D049BB133111EB)
        x ^= x >> np.uint64(31)
    return x


def _items(text: str, measure: str) -> list:
    if measure == "edit":
        return [text[i : i + 3] for i in range(max(1, len(text) - 2))] if text else []
    return tokenize(text)


def branch_keys(relation, pred, banding: BandingConfig) -> list:
    """The reference's Partitioner.keys (partitioning.py:48-78) for one root
    predicate: one key string per tuple."""
    n = len(relation)
    if pred.is_cross_attr:
        return ["x:all"] * n
    k = relation.schema.index_of(pred.lhs_attr)
    numeric = is_numeric_kind(relation.schema.kind_of(pred.lhs_attr))
    col = [rec.values[k] for rec in relation.tuples]
    if pred.comparator == "eq":
        if numeric:
            return [MISSING_KEY if is_missing(v) else f"n:{float(v)!r}" for v in col]
        return [MISSING_KEY if is_missing(v) else f"v:{str(v).strip()}" for v in col]
    # minhash band: hash every distinct item once, then a vectorised min over
    # each tuple's items for every band seed
    rows_items = [[] if is_missing(v) else _items(fold_text(value_text(v)), pred.measure) for v in col]
    vocab: dict = {}
    flat = []
    lens = np.zeros(n, dtype=np.int64)
    for i, items in enumerate(rows_items):
        lens[i] = len(items)
        for it in items:
            flat.append(vocab.setdefault(it, len(vocab)))
    keys = [MISSING_KEY] * n
    if not flat:
        return keys
    item_hash = np.array([stable_hash64(t, banding.seed) for t in vocab], dtype=np.uint64)
    h = item_hash[np.asarray(flat, dtype=np.int64)]
    has = lens > 0
    starts = np.zeros(n, dtype=np.int64)
    np.cumsum(lens[:-1], out=starts[1:])
    sigs = []
    for s in range(banding.seed, banding.seed + banding.rows):
        sigs.append(np.minimum.reduceat(mix64(h, s), starts[has]))
    idx = np.flatnonzero(has)
    for r, i in enumerate(idx):
        keys[i] = "b:" + ":".join(f"{int(sig[r]):x}" for sig in sigs)
    return keys


def root_predicates(path) -> list:
    """Root edges in score order == compile_path's root_slots order, which
    is also derive_partitioners' branch numbering (partitioning.py:81-90)."""
    return [path.predicate_table[s] for s in path.root_slots]


def iter_partitions(relation, path, max_partition_size: int = 512, banding: Optional[BandingConfig] = None):
    """partitioning.py:93-131 over the plan's root edges."""
    banding = banding or BandingConfig()
    roots = root_predicates(path)
    if not roots:
        raise ConfigError("at least one partitioner required")
    if max_partition_size < 1:
        raise ConfigError("max_partition_size must be >= 1")
    pid = 0
    sibling = 0
    order = sorted(range(len(roots)), key=lambda b: roots[b].comparator != "eq")
    for branch in order:
        groups: dict = {}
        for tid, key in enumerate(branch_keys(relation, roots[branch], banding)):
            groups.setdefault(key, []).append(tid)
        for key in sorted(groups):
            refs = groups[key]
            if len(refs) <= max_partition_size:
                yield DataPartition(pid=pid, tuple_refs=tuple(refs), branch_id=branch, key_group=key)
                pid += 1
                continue
            n_parts = -(-len(refs) // max_partition_size)
            sibling += 1
            for sub in range(n_parts):
                yield DataPartition(pid=pid, tuple_refs=tuple(refs[sub::n_parts]), branch_id=branch,
                                    key_group=key, sibling_group=sibling)
                pid += 1


def sibling_pull_pairs(partitions) -> list:
    """partitioning.py:144-157."""
    groups: dict = {}
    for p in partitions:
        if p.sibling_group is not None:
            groups.setdefault(p.sibling_group, []).append(p.pid)
    out = []
    for pids in groups.values():
        pids.sort()
        out += [(pids[i], pids[j]) for i in range(len(pids)) for j in range(i + 1, len(pids))]
    return out


def collect(candidate_sets, rule_ids) -> CandidateSet:
    """pipeline.py:407-421: the union of all rows, deduplicated per (t, s)
    keeping the earliest rule in rule-set order."""
    ts = [cs.arrays for cs in candidate_sets if len(cs)]
    if not ts:
        return CandidateSet(pairs=[], rule_ids=rule_ids, arrays=(np.zeros(0, np.int64),) * 3)
    t = np.concatenate([a[0] for a in ts])
    s = np.concatenate([a[1] for a in ts])
    r = np.concatenate([a[2] for a in ts])
    order = np.lexsort((r, s, t))
    t, s, r = t[order], s[order], r[order]
    keep = np.ones(len(t), dtype=bool)
    keep[1:] = (t[1:] != t[:-1]) | (s[1:] != s[:-1])
    return CandidateSet(arrays=(t[keep], s[keep], r[keep]), rule_ids=rule_ids)


def branch_order(path) -> list:
    """The reference's iteration order over the root edges: equality
    branches first, score order otherwise (partitioning.py:106-110)."""
    roots = root_predicates(path)
    return sorted(range(len(roots)), key=lambda b: roots[b].comparator != "eq")


def rank_keys(keys: list) -> tuple[np.ndarray, list]:
    """Key strings -> int64 ranks in sorted key-string order (the order of
    ``sorted(groups)``), plus the sorted distinct keys."""
    index: dict = {}
    inv = np.fromiter((index.setdefault(k, len(index)) for k in keys), dtype=np.int64, count=len(keys))
    distinct = list(index)
    order = sorted(range(len(distinct)), key=distinct.__getitem__)
    rank = np.empty(len(distinct), dtype=np.int64)
    rank[np.asarray(order, dtype=np.int64)] = np.arange(len(distinct), dtype=np.int64)
    return rank[inv], [distinct[k] for k in order]


def _key_of_value(v, numeric: bool) -> str:
    """The reference's equality key string of one value (partitioning.py:48-78)."""
    if is_missing(v):
        return MISSING_KEY
    return f"n:{float(v)!r}" if numeric else f"v:{str(v).strip()}"


def eq_branch_keys(relation, enc, pred):
    """branch_keys + rank_keys for a same-attribute equality root, from the
    encoding's dictionary codes: the reference key string is formed once per
    DISTINCT value (a representative tuple of each code) instead of once per
    tuple, then ranked; equal codes <=> equal canonical values <=> equal key
    strings (missing: code -1 <=> MISSING_KEY).  Returns (int64 rank per
    tuple, sorted distinct key strings), as rank_keys(branch_keys(...))."""
    enc.slot_for(pred)
    codes = enc.columns[enc.get(("codes", pred.lhs_attr))].data
    numeric = is_numeric_kind(relation.schema.kind_of(pred.lhs_attr))
    present = np.flatnonzero(codes >= 0)
    uniq, first = np.unique(codes[present], return_index=True)
    reps = present[first]
    if hasattr(relation, "column"):
        col = relation.column(pred.lhs_attr)
        vals = [col[int(t)] for t in reps]
    else:
        k = relation.schema.index_of(pred.lhs_attr)
        vals = [relation.tuples[int(t)].values[k] for t in reps]
    keys = [_key_of_value(v, numeric) for v in vals]
    has_missing = len(present) < len(codes)
    distinct = sorted(keys + ([MISSING_KEY] if has_missing else []))
    pos = {key: r for r, key in enumerate(distinct)}
    lut = np.full(int(uniq.max()) + 2 if len(uniq) else 1, -1, dtype=np.int64)
    lut[uniq] = [pos[key] for key in keys]
    ranks = np.where(codes >= 0, lut[np.maximum(codes, 0)], pos.get(MISSING_KEY, -1)).astype(np.int64)
    return ranks, distinct


def branch_ranks(relation, path, b: int, banding: BandingConfig, enc=None):
    """(int64 key rank per tuple, sorted distinct key strings) of branch b:
    from the encoding's codes for a same-attribute equality root (O(distinct
    values) key strings), else from the key strings of every tuple."""
    pred = root_predicates(path)[b]
    if enc is not None and pred.comparator == "eq" and not pred.is_cross_attr and pred.rhs_attr is not None:
        return eq_branch_keys(relation, enc, pred)
    return rank_keys(branch_keys(relation, pred, banding))


def partition_keys(relation, path, banding: Optional[BandingConfig] = None, enc=None):
    """Per branch in iteration order: (branch id, int64 key per tuple, sorted
    distinct key strings).  Equal keys <=> equal reference key strings."""
    banding = banding or BandingConfig()
    out = []
    for b in branch_order(path):
        ranks, distinct = branch_ranks(relation, path, b, banding, enc)
        out.append((b, ranks, distinct))
    return out


class DeviceParts:
    """A partition set resident on one device (rb_parts): the tuple ids of
    every branch sorted into groups and siblings, the partition list, the
    pulls.  ``partitions()`` / ``pulls()`` materialise the reference objects."""

    def __init__(self, handle, ctx, key_groups=None):
        from . import _lib

        self.handle = handle
        self.ctx = ctx
        self.key_groups = key_groups  # branch id -> sorted distinct key strings (exact key_group labels)
        self._fin = weakref.finalize(self, _lib.lib().rb_parts_destroy, handle)
        vals = [_lib.ctypes.c_int64(0) for _ in range(4)]
        _lib.check(_lib.lib().rb_parts_info(handle, *[_lib.ctypes.byref(v) for v in vals]))
        self.n_partitions, self.n_pulls, self.n_refs, self.n_groups = (v.value for v in vals)
        self._host = None

    def close(self) -> None:
        self._fin()

    def host(self):
        """refs and per-entry (base, size, split, rbase, branch, sibling) arrays."""
        if self._host is None:
            from . import _lib

            m = self.n_partitions + self.n_pulls
            refs = np.empty(self.n_refs, dtype=np.int32)
            base, size, split, rbase = (np.empty(m, dtype=np.int64) for _ in range(4))
            branch, sib = np.empty(m, dtype=np.int32), np.empty(m, dtype=np.int32)
            _lib.check(_lib.lib().rb_parts_copy(self.handle, _lib.ptr(refs), _lib.ptr(base), _lib.ptr(size),
                                                _lib.ptr(split), _lib.ptr(rbase), _lib.ptr(branch), _lib.ptr(sib)))
            self._host = (refs, base, size, split, rbase, branch, sib)
        return self._host

    def partitions(self) -> list:
        """DataPartition per partition, pids in order (iter_partitions)."""
        refs, base, size, _, _, branch, sib = self.host()
        out = []
        group_of: dict = {}
        for k in range(self.n_partitions):
            b = int(branch[k])
            key = None
            if self.key_groups is not None:
                # groups come in key order: count the distinct groups seen in this branch
                g = group_of.setdefault(b, [-1, -1])
                if sib[k] == 0 or sib[k] != g[1]:
                    g[0] += 1
                g[1] = int(sib[k]) if sib[k] else -1
                key = self.key_groups[b][g[0]]
            out.append(DataPartition(pid=k, tuple_refs=tuple(refs[base[k]:base[k] + size[k]].tolist()), branch_id=b,
                                     key_group=key, sibling_group=int(sib[k]) if sib[k] else None))
        return out

    def pulls(self) -> list:
        """(pid_a, pid_b) per pull, as sibling_pull_pairs."""
        _, base, _, split, rbase, _, _ = self.host()
        start_pid = {int(base[k]): k for k in range(self.n_partitions)}
        return [(start_pid[int(base[k])], start_pid[int(rbase[k])])
                for k in range(self.n_partitions, self.n_partitions + self.n_pulls)]


def implied_root_slots(path, branch_ids) -> list:
    """Per branch: the path slot its partition key implies for every pair of
    a group -- the root slot of a same-attribute equality edge (equal
    canonical keys <=> equal codes <=> the slot holds, outside the missing
    group) -- or -1 (minhash bands, cross-attribute keys)."""
    out = []
    for b in branch_ids:
        s = path.root_slots[b]
        p = path.predicate_table[s]
        out.append(int(s) if p.comparator == "eq" and not p.is_cross_attr and p.rhs_attr is not None else -1)
    return out


def partition_on_device(prog, *, keys=None, code_cols=None, branch_ids, max_partition_size: int, pulls: bool,
                        key_groups=None) -> DeviceParts:
    """rb_partition / rb_partition_codes over the program's relation.
    ``keys``: int64 array (branches, n) in iteration order; ``code_cols``:
    the relation's codes columns, one per branch."""
    from . import _lib

    if max_partition_size < 1:
        raise ConfigError("max_partition_size must be >= 1")
    L = _lib.lib()
    h = _lib.c_vp()
    bids = np.ascontiguousarray(branch_ids, dtype=np.int32)
    flags = _lib.RB_PART_PULLS if pulls else 0
    if keys is not None:
        k = np.ascontiguousarray(keys, dtype=np.int64)
        _lib.check(L.rb_partition(prog.ctx.handle, prog.drel.handle, _lib.ptr(k), _lib.ptr(bids), len(bids),
                                  int(max_partition_size), flags, _lib.ctypes.byref(h)))
    else:
        cols = np.ascontiguousarray(code_cols, dtype=np.int32)
        _lib.check(L.rb_partition_codes(prog.ctx.handle, prog.drel.handle, _lib.ptr(cols), _lib.ptr(bids), len(bids),
                                        int(max_partition_size), flags, _lib.ctypes.byref(h)))
    parts = DeviceParts(h, prog.ctx, key_groups)
    roots = np.ascontiguousarray(implied_root_slots(prog.path, list(bids)), dtype=np.int32)
    first_missing = None
    if keys is not None:  # ranked key strings: the missing key sorts first when a branch has one
        first_missing = np.array([1 if key_groups is None or not key_groups.get(int(b)) else
                                  int(key_groups[int(b)][0] == MISSING_KEY) for b in bids], dtype=np.uint8)
    _lib.check(L.rb_parts_set_roots(h, _lib.ptr(roots), _lib.ptr(first_missing), len(roots)))
    return parts


@dataclass
class PipelineResult:
    """pipeline.py:212-220 (candidates, timings, assignment, n_partitions,
    device_busy_s, plan) plus the device partition set."""

    candidates: CandidateSet
    timings: dict
    assignment: dict
    n_partitions: int
    device_busy_s: dict
    plan: object = None
    parts: object = None  # DeviceParts of the first device (partitions() / pulls())

    @property
    def partitions(self) -> list:
        return [] if self.parts is None else self.parts.partitions()


def _cuda_devices(devices, pipe_cfg) -> list:
    """CUDA ordinals: ints as given; the reference's simulated Device
    objects map onto the visible GPUs by device_id."""
    if not devices:
        return list(pipe_cfg.devices)
    out = []
    for d in devices:
        out.append(int(getattr(d, "device_id", d)))
    return out


class ResidentPipeline:
    """pipeline_run's device stages over a relation already resident on one
    GPU (a ``PathProgram`` and its ``DeviceRelation``): partition, execute
    this rank's LPT share of the units, collect; with ``world > 1`` the
    collected rows are then exchanged by tuple-id range between the ranks
    (``distributed.exchange_rows``, one NCCL all-to-all) and collected once
    more, so rank r ends with the final candidate rows whose t lies in its
    range -- the ranks' shards in rank order are the collected set.

    ``step()`` is one pass of the hot path (BASELINE config 4 (i)); every
    stage is timed with CUDA events on the context's stream (the bench binds
    the context to torch's current stream)."""

    def __init__(self, prog, *, keys=None, code_cols=None, branch_ids, max_partition_size: int, pulls: bool,
                 flags: int, key_groups=None):
        self.prog = prog
        self.keys = keys
        self.code_cols = code_cols
        self.branch_ids = list(branch_ids)
        self.maxp = int(max_partition_size)
        self.pulls = bool(pulls)
        self.flags = int(flags)
        self.key_groups = key_groups
        self.n_tuples = prog.enc.n
        self.n_rules = max(1, len(prog.rule_ids))
        self.res = None  # the last single-rank step's DeviceResult (its rows are views)
        self.parts = None

    def close(self) -> None:
        if self.res is not None:
            self.res.close()
            self.res = None
        if self.parts is not None:
            self.parts.close()
            self.parts = None

    def step(self, rank: int = 0, world: int = 1, group=None, events: bool = False, keep_parts: bool = False):
        """-> (rows, stats, stage_ms).  ``rows``: (t, s, rule) int32 device
        tensors of this rank's collected shard (at world 1: views of the
        result buffers, valid until the next step() or close()); the rows
        are exchanged between the ranks only when ``group`` is given (one
        process per GPU); without it the caller merges the ranks' rows
        (several devices driven from one process); ``stats``: the run's rb_stats
        (this rank's units); ``stage_ms``: partition / execute / collect /
        exchange milliseconds (CUDA events when ``events``, else host clock
        around the stage; every stage ends on a host sync).  ``keep_parts``:
        the partition set stays alive as ``self.parts`` (DeviceParts)."""
        import torch

        dev = torch.device("cuda", self.prog.ctx.device)
        marks = []

        def mark():
            if events:
                e = torch.cuda.Event(enable_timing=True)
                e.record(torch.cuda.current_stream(dev))
                marks.append(e)
            else:
                marks.append(time.perf_counter())

        mark()
        parts = partition_on_device(self.prog, keys=self.keys, code_cols=self.code_cols, branch_ids=self.branch_ids,
                                    max_partition_size=self.maxp, pulls=self.pulls, key_groups=self.key_groups)
        mark()
        res = self.prog.run_parts(parts, self.flags, rank, world)
        st = res.stats()
        if self.parts is not None:
            self.parts.close()
            self.parts = None
        if keep_parts:
            self.parts = parts
        else:
            parts.close()
        mark()
        res.collect(self.n_tuples, self.n_rules)
        if self.res is not None:
            self.res.close()
        self.res = None
        exchange = group is not None and world > 1
        rows = res.torch_views()
        if not exchange:  # the rows stay in the result's buffers: views, valid until the next step / close()
            self.res = res
        mark()
        if exchange:
            from .distributed import exchange_rows

            rows = exchange_rows(rows, self.n_tuples, group)  # packed copies of the views
            torch.cuda.current_stream(dev).synchronize()  # before the library frees the viewed buffers
            res.close()
            rows = collect_device_rows(rows, self.n_tuples, self.n_rules, self.prog.ctx)
        mark()
        if events:
            torch.cuda.current_stream(dev).synchronize()
            ms = [marks[k].elapsed_time(marks[k + 1]) for k in range(len(marks) - 1)]
        else:
            ms = [1e3 * (marks[k + 1] - marks[k]) for k in range(len(marks) - 1)]
        stage_ms = dict(zip(("partition", "execute", "collect", "exchange"), ms))
        return rows, st, stage_ms


def collect_device_rows(rows, n_tuples: int, n_rules: int, ctx):
    """rb_collect_device over (t, s, rule) int32 device tensors -> new
    tensors (sorted by (t, s), smallest rule per (t, s))."""
    import torch

    from . import _lib

    k = int(rows[0].shape[0])
    dev = rows[0].device
    out = [torch.empty(max(1, k), dtype=torch.int32, device=dev) for _ in range(3)]
    if k == 0:
        return tuple(x[:0] for x in out)
    torch.cuda.current_stream(dev).synchronize()  # the inputs precede the library's stream
    cnt = _lib.ctypes.c_int64(0)
    _lib.check(_lib.lib().rb_collect_device(ctx.handle, *[_lib.c_vp(x.data_ptr()) for x in rows], k, n_tuples,
                                            n_rules, *[_lib.c_vp(x.data_ptr()) for x in out], _lib.ctypes.byref(cnt)))
    return tuple(x[: cnt.value] for x in out)


def _merge_runs(runs: list, n_tuples: int, n_rules: int, device: int):
    """Collected row runs of several devices -> one collected set (host
    arrays): concatenated and collected once more on ``device``."""
    if len(runs) == 1:
        return runs[0]
    import torch

    from . import _lib
    from .engine import context

    total = sum(len(r[0]) for r in runs)
    if total == 0:
        return tuple(np.zeros(0, np.int32) for _ in range(3))
    dev = torch.device("cuda", device)
    cols = [torch.from_numpy(np.concatenate([r[c] for r in runs])).to(dev) for c in range(3)]
    out = collect_device_rows(cols, n_tuples, n_rules, context(device))
    return tuple(x.cpu().numpy() for x in out)


def _device_stage(dev: int, enc, path, compiled, keys, code_cols, branch_ids, maxp: int, pulls: bool, cfg,
                  rank: int, world: int, key_groups, timings: dict, group=None, out=None):
    """One device: upload, then ResidentPipeline.step (partition, this
    rank's share, collect; exchange when ``group`` spans several ranks).
    Returns (host rows of the rank, rb_stats, DeviceParts)."""
    from .engine import DeviceRelation, PathProgram, context

    t0 = time.perf_counter()
    ctx = context(dev)
    drel = DeviceRelation(ctx, enc)
    prog = PathProgram(path, enc, compiled=compiled, drel=drel)
    t1 = time.perf_counter()
    rp = ResidentPipeline(prog, keys=keys, code_cols=code_cols, branch_ids=branch_ids, max_partition_size=maxp,
                          pulls=pulls, flags=cfg.flags(), key_groups=key_groups)
    rows, st, ms = rp.step(rank, world, group, keep_parts=True)
    t2 = time.perf_counter()
    k = int(rows[0].shape[0])
    if out is not None and all(len(a) >= k and a.dtype == np.int32 and a.flags["C_CONTIGUOUS"] for a in out):
        import torch

        host = tuple(a[:k] for a in out)  # caller's (pinned) host buffers: D2H at link speed
        for h, x in zip(host, rows):
            if k:
                torch.from_numpy(h).copy_(x)
    else:
        host = tuple(x.cpu().numpy() for x in rows)
    if rp.res is not None:  # the rows were views of it
        rp.res.close()
        rp.res = None
    t3 = time.perf_counter()
    prog.close()
    drel.close()
    timings.update(upload_s=t1 - t0, partition_s=ms["partition"] / 1e3, execute_s=ms["execute"] / 1e3,
                   collect_s=ms["collect"] / 1e3, exchange_s=ms["exchange"] / 1e3, d2h_s=t3 - t2)
    return host, st, rp.parts


def run_pipeline_encoded(enc, path, pipe_cfg: Optional[PipelineConfig] = None,
                         engine_cfg: Optional[EngineConfig] = None, *, keys=None, code_cols=None, branch_ids=None,
                         devices=None, reg=None, key_groups=None, group=None, compiled=None,
                         out=None) -> PipelineResult:
    """The device pipeline over an encoded relation: partition (``keys``
    int64 (branches, n) or eq-root ``code_cols``), execute, collect.

    * ``group`` None: every device in ``devices`` runs its LPT share of the
      units from a host thread of this process; the rows are merged and
      collected once more on the first device.
    * ``group`` a torch.distributed process group (one process per GPU, this
      process on ``torch.cuda.current_device()``): this rank runs its share,
      the rows are exchanged by tuple-id range over the group (NCCL
      all-to-all) and collected; the result holds this rank's shard (t in
      ``distributed.t_bounds(n, world)[rank:rank + 2]``).  Collective.
    ``out``: optional (t, s, rule) int32 host arrays (e.g. pinned) the rows
    are copied into when they fit (one device only)."""
    from .encode import compile_program

    pipe_cfg = pipe_cfg or PipelineConfig()
    engine_cfg = engine_cfg or EngineConfig(num_blocks=1)
    n = enc.n
    if compiled is None:
        compiled = compile_program(path, enc, reg)
    threshold = pipe_cfg.single_partition_threshold
    if threshold is None:
        threshold = pipe_cfg.max_partition_size
    maxp = pipe_cfg.max_partition_size
    if n <= threshold:  # one partition of every tuple (pipeline.py:282-286)
        keys, code_cols, branch_ids, key_groups = np.zeros((1, n), np.int64), None, [0], None
        maxp = max(1, n)
    if branch_ids is None:
        branch_ids = branch_order(path)
    n_rules = max(1, len(path.rule_ids))
    wall0 = time.perf_counter()
    if group is not None:
        import torch
        import torch.distributed as dist

        devs = [torch.cuda.current_device()]
        rank, world = dist.get_rank(group), dist.get_world_size(group)
    else:
        devs = _cuda_devices(devices, pipe_cfg)
        rank, world = 0, len(devs)
    per_dev: list = [None] * len(devs)
    errors: list = []

    def work(k: int):
        try:
            tm: dict = {}
            rows, st, parts = _device_stage(devs[k], enc, path, compiled, keys, code_cols, branch_ids, maxp,
                                            pipe_cfg.enable_pulls, engine_cfg, rank + k, world, key_groups, tm, group,
                                            out if len(devs) == 1 else None)
            if k:
                parts.close()
                parts = None
            per_dev[k] = (rows, st, tm, parts)
        except BaseException as exc:  # surfaced below
            errors.append(exc)

    if len(devs) == 1:
        work(0)
    else:
        threads = [threading.Thread(target=work, args=(k,), name=f"rb-pipeline-gpu{devs[k]}") for k in range(len(devs))]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
    if errors:
        raise errors[0]
    t0 = time.perf_counter()
    if group is None:
        t, s, r = _merge_runs([x[0] for x in per_dev], n, n_rules, devs[0])
    else:
        t, s, r = per_dev[0][0]
    merge_s = time.perf_counter() - t0
    keys_t = ("upload_s", "partition_s", "execute_s", "collect_s", "exchange_s", "d2h_s")
    timings = {k: max(x[2][k] for x in per_dev) for k in keys_t}
    timings["collect_s"] += merge_s
    timings["total_s"] = time.perf_counter() - wall0
    stats = [x[1] for x in per_dev]
    from .engine import BlockStats

    blocks = [BlockStats(block_id=rank + k, comparisons=int(st.comparisons), survivors=int(st.survivors),
                         emitted=int(st.emitted), busy_s=st.kernel_ms / 1e3,
                         slot_evals=np.array(st.slot_evals[: len(path.predicate_table)], dtype=np.int64))
              for k, st in enumerate(stats)]
    cand = CandidateSet(arrays=(t, s, r),  # int32 as copied back (no host widening pass)
                        rule_ids=list(path.rule_ids),
                        stats=RunStats(blocks=blocks, wall_s=timings["total_s"],
                                       kernel_ms=sum(st.kernel_ms for st in stats),
                                       launches=sum(int(st.launches) for st in stats)))
    parts = per_dev[0][3]
    return PipelineResult(candidates=cand, timings=timings, assignment={}, n_partitions=int(parts.n_partitions),
                          device_busy_s={devs[k]: per_dev[k][1].kernel_ms / 1e3 for k in range(len(devs))},
                          plan=None, parts=parts)


def pipeline_run(relation, rules, pipe_cfg: Optional[PipelineConfig] = None,
                 engine_cfg: Optional[EngineConfig] = None, devices=None, planner_cfg=None, plan=None, reg=None,
                 encoded=None) -> PipelineResult:
    """The reference's pipeline_run (pipeline.py:245-433) on the GPU(s):
    partition, evaluate every partition (and sibling pull), collect.

    ``rules`` is the RuleSet (with ``plan``, a PlanBundle or anything with a
    ``.path``, frozen as the reference's ``plan=``) or directly an
    ExecutionPath.  Without a plan, a data-aware plan is derived from sampled
    selectivities (plan generation itself is outside this path).  ``devices``:
    CUDA ordinals or the reference's Device objects (by device_id)."""
    from .encode import RelationEncoding
    from .engine import _encoding_for

    pipe_cfg = pipe_cfg or PipelineConfig()
    engine_cfg = engine_cfg or EngineConfig(num_blocks=1)
    t0 = time.perf_counter()
    if plan is not None:
        path = getattr(plan, "path", plan)
    elif hasattr(rules, "predicate_table"):
        path = rules
    else:
        from .synth import data_aware_plan

        path = None
    plan_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    enc = _encoding_for(relation, encoded)
    if path is None:
        path = data_aware_plan(RelationEncoding(relation).prepare(list(_universe(rules))), rules)
    if isinstance(enc, RelationEncoding):
        enc.prepare(list(path.predicate_table))
    encode_s = time.perf_counter() - t0
    threshold = pipe_cfg.single_partition_threshold
    if threshold is None:
        threshold = pipe_cfg.max_partition_size
    if len(relation) <= threshold:
        res = run_pipeline_encoded(enc, path, pipe_cfg, engine_cfg, devices=devices, reg=reg)
        res.timings.update(keys_s=0.0)
    else:
        res = _streamed_pipeline(relation, enc, path, pipe_cfg, engine_cfg, devices, reg)
    res.timings.update(plan_s=plan_s, encode_s=encode_s)
    res.timings["total_s"] += plan_s + encode_s
    res.plan = plan
    return res


class _BranchParts:
    """The partition set of a streamed pipeline run: one DeviceParts per
    branch (each numbered from 0), read back as the reference's single pid /
    sibling-group sequence (iter_partitions order across branches)."""

    def __init__(self, parts: list):
        self.parts = parts
        self.n_partitions = sum(int(p.n_partitions) for p in parts)
        self.n_pulls = sum(int(p.n_pulls) for p in parts)

    def close(self) -> None:
        for p in self.parts:
            p.close()

    def partitions(self) -> list:
        out, pid0, sib0 = [], 0, 0
        for dp in self.parts:
            got = dp.partitions()
            for p in got:
                out.append(DataPartition(pid=p.pid + pid0, tuple_refs=p.tuple_refs, branch_id=p.branch_id,
                                         key_group=p.key_group,
                                         sibling_group=None if p.sibling_group is None else p.sibling_group + sib0))
            pid0 += len(got)
            sib0 += max([p.sibling_group or 0 for p in got], default=0)
        return out

    def pulls(self) -> list:
        out, pid0 = [], 0
        for dp in self.parts:
            out += [(a + pid0, b + pid0) for a, b in dp.pulls()]
            pid0 += int(dp.n_partitions)
        return out


def _streamed_pipeline(relation, enc, path, pipe_cfg, engine_cfg, devices, reg) -> PipelineResult:
    """pipeline_run over hash partitions, branch by branch: the host computes
    the next branch's partition keys (key strings, minhash bands) while every
    device partitions and evaluates its LPT share of the previous branch --
    the reference's overlapped partition / execute stages (pipeline.py:
    282-283, 352-386).  Each device then collects its rows once; the devices'
    collected runs are merged and collected on the first."""
    import queue

    from .encode import compile_program

    devs = _cuda_devices(devices, pipe_cfg)
    compiled = compile_program(path, enc, reg)
    roots = root_predicates(path)
    n, n_rules = enc.n, max(1, len(path.rule_ids))
    flags = engine_cfg.flags()
    wall0 = time.perf_counter()
    queues = [queue.Queue() for _ in devs]
    per_dev = [{"host": None, "stats": [], "parts": [], "tm": dict(partition_s=0.0, execute_s=0.0, collect_s=0.0,
                                                                  upload_s=0.0, d2h_s=0.0, exchange_s=0.0)}
               for _ in devs]
    errors: list = []

    def worker(k: int):
        import torch

        from .engine import DeviceRelation, PathProgram, context

        d = per_dev[k]
        results = []
        try:
            t0 = time.perf_counter()
            ctx = context(devs[k])
            drel = DeviceRelation(ctx, enc)
            prog = PathProgram(path, enc, compiled=compiled, drel=drel)
            d["tm"]["upload_s"] += time.perf_counter() - t0
            while True:
                item = queues[k].get()
                if item is None:
                    break
                b, keys_b, groups_b = item
                t0 = time.perf_counter()
                parts = partition_on_device(prog, keys=keys_b[None, :], branch_ids=[b],
                                            max_partition_size=pipe_cfg.max_partition_size,
                                            pulls=pipe_cfg.enable_pulls, key_groups={b: groups_b})
                t1 = time.perf_counter()
                res = prog.run_parts(parts, flags, k, len(devs))
                d["stats"].append(res.stats())
                results.append(res)
                if k == 0:
                    d["parts"].append(parts)
                else:
                    parts.close()
                d["tm"]["partition_s"] += t1 - t0
                d["tm"]["execute_s"] += time.perf_counter() - t1
            t0 = time.perf_counter()
            views = [r.torch_views() for r in results]
            rows = tuple(torch.cat([v[c] for v in views]) if views else torch.empty(0, dtype=torch.int32,
                                                                                    device=f"cuda:{devs[k]}")
                         for c in range(3))
            rows = collect_device_rows(rows, n, n_rules, ctx)
            d["tm"]["collect_s"] += time.perf_counter() - t0
            t0 = time.perf_counter()
            d["host"] = tuple(x.cpu().numpy() for x in rows)
            d["tm"]["d2h_s"] += time.perf_counter() - t0
            prog.close()
            drel.close()
        except BaseException as exc:  # surfaced below
            errors.append(exc)
            while queues[k].get() is not None:  # drain: the producer must not block
                pass
        finally:
            for r in results:
                r.close()

    threads = [threading.Thread(target=worker, args=(k,), name=f"rb-pipeline-gpu{devs[k]}") for k in range(len(devs))]
    for t in threads:
        t.start()
    keys_s = 0.0
    try:
        for b in branch_order(path):  # host keys of branch b overlap the devices' work on branch b - 1
            t0 = time.perf_counter()
            ranks, distinct = branch_ranks(relation, path, b, pipe_cfg.banding, enc)
            keys_s += time.perf_counter() - t0
            for q in queues:
                q.put((b, ranks, distinct))
    finally:
        for q in queues:
            q.put(None)
        for t in threads:
            t.join()
    if errors:
        for p in per_dev[0]["parts"]:
            p.close()
        raise errors[0]
    t0 = time.perf_counter()
    t, s, r = _merge_runs([d["host"] for d in per_dev], n, n_rules, devs[0])
    merge_s = time.perf_counter() - t0
    timings = {key: max(d["tm"][key] for d in per_dev) for key in per_dev[0]["tm"]}
    timings["collect_s"] += merge_s
    timings["keys_s"] = keys_s
    timings["total_s"] = time.perf_counter() - wall0
    from .engine import BlockStats

    blocks, kernel_ms, launches = [], 0.0, 0
    for k, d in enumerate(per_dev):
        st = d["stats"]
        blocks.append(BlockStats(block_id=k, comparisons=sum(int(x.comparisons) for x in st),
                                 survivors=sum(int(x.survivors) for x in st), emitted=sum(int(x.emitted) for x in st),
                                 busy_s=sum(x.kernel_ms for x in st) / 1e3,
                                 slot_evals=np.sum([np.array(x.slot_evals[: len(path.predicate_table)], dtype=np.int64)
                                                    for x in st], axis=0) if st else
                                 np.zeros(len(path.predicate_table), dtype=np.int64)))
        kernel_ms += sum(x.kernel_ms for x in st)
        launches += sum(int(x.launches) for x in st)
    cand = CandidateSet(arrays=(t, s, r), rule_ids=list(path.rule_ids),
                        stats=RunStats(blocks=blocks, wall_s=timings["total_s"], kernel_ms=kernel_ms,
                                       launches=launches))
    parts = _BranchParts(per_dev[0]["parts"])
    return PipelineResult(candidates=cand, timings=timings, assignment={}, n_partitions=parts.n_partitions,
                          device_busy_s={devs[k]: per_dev[k]["tm"]["execute_s"] for k in range(len(devs))},
                          plan=None, parts=parts)


def _universe(rules):
    from .rules import predicate_universe

    return predicate_universe(rules)
