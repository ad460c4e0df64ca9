"""Multi-GPU execution of many partitions: static cost-balanced placement
with work stealing, and copy/compute overlap through two streams per GPU.

Reference counterparts (pkg/src/ruleblock/):
  * the device fleet and per-device worker processes   pipeline.py:39-48, 177-209
  * CHBL placement / the live scheduler                 pipeline.py:92-157
  * inter-interval stealing                            engine.py:163-184
  * the async staged pipeline                           pipeline.py:352-386
  * the collector's union of candidate rows             pipeline.py:407-421

Here a *unit* is either a batch of small partitions / cross blocks (one
``rb_run_batch`` launch) or an outer-row shard of one large partition
(``rb_run_partition_rows``).  Units are placed statically on the devices by
longest-processing-time on their pair counts; a device whose own queue runs
dry steals from the back of the most loaded device's queue.  Each device runs
``workers_per_device`` host threads, each with its own CUDA context stream,
so the host-to-device copy and launch of one unit overlaps the kernel of the
other (ctypes releases the GIL for the whole device call).  No data-path
collective: devices exchange nothing; the caller merges the per-partition
results.
"""

from __future__ import annotations

import threading
import time
from collections import deque
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from .engine import (
    CandidateSet,
    EngineConfig,
    PathProgram,
    RunStats,
    _batch,
    _candidates,
    _encoding_for,
    _refs_array,
    split_rows_by_pairs,
)
from .encode import RelationEncoding, compile_program
from .errors import ConfigError, SchemaError


@dataclass
class Unit:
    """One schedulable piece of work."""

    uid: int
    cost: int  # pairs it evaluates
    blocks: list = field(default_factory=list)  # [(block index, refs, split)] for batch units
    shard: Optional[tuple] = None  # (block index, refs, row_lo, row_hi) for a row shard


def pair_count(n: int, split: int, symmetric: bool) -> int:
    if split >= 0:
        return split * (n - split)
    return n * (n - 1) // 2 if symmetric else n * (n - 1)


def make_units(blocks, symmetric: bool, batch_pairs: int, shard_pairs: int) -> list:
    """blocks: [(refs int32, split)].  Small blocks are packed into batches of
    about `batch_pairs` pairs; a partition larger than `shard_pairs` is cut
    into equal-pair outer-row shards."""
    units: list = []
    cur: list = []
    cur_cost = 0
    order = sorted(range(len(blocks)), key=lambda k: -pair_count(len(blocks[k][0]), blocks[k][1], symmetric))
    for k in order:
        refs, split = blocks[k]
        c = pair_count(len(refs), split, symmetric)
        if c == 0:
            continue
        if split < 0 and c > shard_pairs:
            parts = max(2, -(-c // shard_pairs))
            for lo, hi in split_rows_by_pairs(len(refs), parts, symmetric):
                if hi > lo:
                    sc = (hi - lo) * len(refs) - (hi * (hi + 1) - lo * (lo + 1)) // 2 if symmetric else (hi - lo) * (len(refs) - 1)
                    units.append(Unit(len(units), sc, shard=(k, refs, lo, hi)))
            continue
        cur.append((k, refs, split))
        cur_cost += c
        if cur_cost >= batch_pairs:
            units.append(Unit(len(units), cur_cost, blocks=cur))
            cur, cur_cost = [], 0
    if cur:
        units.append(Unit(len(units), cur_cost, blocks=cur))
    return units


class StealingQueues:
    """Static LPT placement over devices plus stealing from the back of the
    most loaded queue."""

    def __init__(self, units: list, n_devices: int):
        self.queues = [deque() for _ in range(n_devices)]
        self.load = [0] * n_devices
        for u in sorted(units, key=lambda u: -u.cost):
            d = min(range(n_devices), key=lambda k: self.load[k])
            self.queues[d].append(u)
            self.load[d] += u.cost
        self.lock = threading.Lock()
        self.steals = [0] * n_devices

    def next(self, device: int) -> Optional[Unit]:
        with self.lock:
            if self.queues[device]:
                return self.queues[device].popleft()
            victim = max(range(len(self.queues)), key=lambda k: sum(u.cost for u in self.queues[k]))
            if self.queues[victim]:
                self.steals[device] += 1
                return self.queues[victim].pop()
            return None


class MultiDeviceEngine:
    """Evaluate one path over many partitions on several GPUs.

    ``devices`` lists CUDA device ordinals (repeat one to test on a single
    GPU).  The encoded relation is uploaded once per device and shared by
    that device's worker threads; each worker runs its own program on its
    own context (stream), so the H2D and launch of one unit overlap the
    kernel of another."""

    def __init__(self, relation, path, devices=(0,), reg=None, encoded=None, workers_per_device: int = 2,
                 batch_pairs: int = 1 << 30, shard_pairs: int = 1 << 34):
        if not devices:
            raise ConfigError("at least one device is required")
        self.relation = relation
        self.path = path
        self.devices = list(devices)
        self.workers_per_device = max(1, int(workers_per_device))
        self.batch_pairs = batch_pairs
        self.shard_pairs = shard_pairs
        enc = _encoding_for(relation, encoded)
        if isinstance(enc, RelationEncoding):
            enc.prepare(list(path.predicate_table))
        self.enc = enc
        self.compiled = compile_program(path, enc, reg)
        self.last_steals: list = []
        self.last_busy_s: list = []
        self._rels: dict = {}  # device -> (owning context, DeviceRelation)
        self._rel_lock = threading.Lock()

    def _relation(self, device: int):
        """One uploaded relation per device, shared by its workers' contexts."""
        with self._rel_lock:
            if device not in self._rels:
                from .engine import Context, DeviceRelation

                owner = Context(device)
                self._rels[device] = (owner, DeviceRelation(owner, self.enc))
            return self._rels[device][1]

    def _program(self, device: int, cache: dict) -> PathProgram:
        if "prog" not in cache:
            from .engine import Context

            ctx = Context(device)  # a private context (stream) for this worker thread
            cache["prog"] = PathProgram(self.path, self.enc, compiled=self.compiled, drel=self._relation(device),
                                        ctx=ctx)
        return cache["prog"]

    def run(self, blocks, cfg: Optional[EngineConfig] = None) -> list:
        """blocks: [(refs, split)] with split = -1 for a partition, else the
        size of the left side of a cross block.  Returns a CandidateSet per
        block."""
        cfg = EngineConfig.of(cfg)
        units = make_units(blocks, cfg.symmetric_mode, self.batch_pairs, self.shard_pairs)
        queues = StealingQueues(units, len(self.devices))
        results: dict = {}
        errors: list = []
        busy = [0.0] * len(self.devices)
        lock = threading.Lock()

        def worker(d: int):
            cache: dict = {}
            try:
                while True:
                    u = queues.next(d)
                    if u is None:
                        return
                    t0 = time.perf_counter()
                    prog = self._program(self.devices[d], cache)
                    if u.shard is not None:
                        k, refs, lo, hi = u.shard
                        rows, st = prog.run_raw(refs, len(refs), cfg.flags(), row_lo=lo, row_hi=hi)
                        cs = _candidates(prog, rows, st, cfg, hi - lo, time.perf_counter() - t0)
                        with lock:
                            results.setdefault(k, []).append(cs)
                    else:
                        out = _batch(prog, [(refs, split) for _, refs, split in u.blocks], cfg)
                        with lock:
                            for (k, _, _), cs in zip(u.blocks, out):
                                results.setdefault(k, []).append(cs)
                    with lock:
                        busy[d] += time.perf_counter() - t0
            except BaseException as exc:  # surfaced to the caller below
                with lock:
                    errors.append(exc)

        threads = [threading.Thread(target=worker, args=(d,), name=f"rb-gpu{self.devices[d]}-w{w}", daemon=True)
                   for d in range(len(self.devices)) for w in range(self.workers_per_device)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        if errors:
            raise errors[0]
        self.last_steals = list(queues.steals)
        self.last_busy_s = busy
        out = []
        for k, (refs, split) in enumerate(blocks):
            parts = results.get(k, [])
            if not parts:
                out.append(CandidateSet(pairs=[]))
            elif len(parts) == 1:
                out.append(parts[0])
            else:
                out.append(merge_shards(parts, cfg))
        return out

    def run_partitions(self, partitions, cfg: Optional[EngineConfig] = None) -> list:
        blocks = [(_refs_array(p), -1) if p is not None and len(p.tuple_refs) else (np.zeros(0, np.int32), -1)
                  for p in partitions]
        return self.run(blocks, cfg)

    def run_crosses(self, pairs, cfg: Optional[EngineConfig] = None) -> list:
        blocks = []
        for left, right in pairs:
            lr, rr = _refs_array(left), _refs_array(right)
            both = np.concatenate([lr, rr])
            if len(np.unique(both)) != len(both):
                raise SchemaError("partition -1 has duplicate tuple refs")
            blocks.append((both, len(lr)))
        return self.run(blocks, cfg)


def merge_shards(parts: list, cfg: EngineConfig) -> CandidateSet:
    """Union of the outer-row shards of one partition: disjoint pair sets,
    so rows simply concatenate; statistics add up."""
    t = np.concatenate([p.arrays[0] for p in parts])
    s = np.concatenate([p.arrays[1] for p in parts])
    r = np.concatenate([p.arrays[2] for p in parts])
    blocks = [b for p in parts for b in p.stats.blocks]
    stats = RunStats(blocks=blocks, wall_s=max(p.stats.wall_s for p in parts),
                     n_intervals=sum(p.stats.n_intervals for p in parts),
                     kernel_ms=sum(p.stats.kernel_ms for p in parts), launches=sum(p.stats.launches for p in parts),
                     specialized=all(p.stats.specialized for p in parts))
    return CandidateSet(stats=stats, arrays=(t, s, r), rule_ids=parts[0]._rule_ids)
