"""The callers on either side of the path: plan-derived partitioning, the
device run over all partitions and pulls, and the collect step.

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
(pids, refs, branches, sibling groups) are identical too.  The heavy part --
minhash over every tuple's items -- is vectorised; the evaluation of all
partitions runs batched on the GPU(s) through scheduler.MultiDeviceEngine.
"""

from __future__ import annotations

import hashlib
import time
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
    max_partition_size: int = 512
    enable_pulls: bool = False
    banding: BandingConfig = field(default_factory=BandingConfig)
    single_partition_threshold: Optional[int] = None  # None: follows max_partition_size
    devices: tuple = (0,)
    workers_per_device: int = 2


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


@dataclass
class PipelineResult:
    candidates: CandidateSet
    timings: dict
    n_partitions: int
    partitions: list


def pipeline_run(relation, path, pipe_cfg: Optional[PipelineConfig] = None,
                 engine_cfg: Optional[EngineConfig] = None, reg=None, encoded=None) -> PipelineResult:
    """The reference's pipeline_run (pipeline.py:245-433) on a frozen path:
    partition, evaluate every partition (and sibling pull) on the GPU(s),
    collect.  Candidate sets equal the reference's for the same plan."""
    from .scheduler import MultiDeviceEngine

    pipe_cfg = pipe_cfg or PipelineConfig()
    engine_cfg = engine_cfg or EngineConfig(num_blocks=1)
    timings: dict = {}
    wall0 = time.perf_counter()
    t0 = time.perf_counter()
    threshold = pipe_cfg.single_partition_threshold
    if threshold is None:
        threshold = pipe_cfg.max_partition_size
    if len(relation) <= threshold:
        partitions = [DataPartition(pid=0, tuple_refs=tuple(range(len(relation))))]
    else:
        partitions = list(iter_partitions(relation, path, pipe_cfg.max_partition_size, pipe_cfg.banding))
    timings["partition_s"] = time.perf_counter() - t0

    t0 = time.perf_counter()
    eng = MultiDeviceEngine(relation, path, devices=pipe_cfg.devices, reg=reg, encoded=encoded,
                            workers_per_device=pipe_cfg.workers_per_device)
    work = [p for p in partitions if len(p.tuple_refs) > 1 or not engine_cfg.symmetric_mode]
    results = eng.run_partitions(work, engine_cfg)
    if pipe_cfg.enable_pulls:
        by_pid = {p.pid: p for p in partitions}
        pulls = [(by_pid[a], by_pid[b]) for a, b in sibling_pull_pairs(partitions)]
        results += eng.run_crosses(pulls, engine_cfg) if pulls else []
    timings["execute_s"] = time.perf_counter() - t0

    t0 = time.perf_counter()
    cand = collect(results, list(path.rule_ids))
    timings["collect_s"] = time.perf_counter() - t0
    timings["total_s"] = time.perf_counter() - wall0
    cand.stats = RunStats(blocks=[b for cs in results for b in cs.stats.blocks], wall_s=timings["total_s"])
    return PipelineResult(candidates=cand, timings=timings, n_partitions=len(partitions), partitions=partitions)
