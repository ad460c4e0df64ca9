"""Multi-device scheduling: unit construction, LPT placement and work
stealing (CPU), and the threaded multi-GPU engine (GPU, two workers per
device and a repeated device ordinal to emulate several GPUs)."""

import random
import threading
import time

import numpy as np
import pytest

import goldens
from paper_2410_04349_b200 import DataPartition, EngineConfig, run_partition
from paper_2410_04349_b200.scheduler import MultiDeviceEngine, StealingQueues, Unit, make_units, pair_count


def test_make_units_packs_small_and_shards_large():
    rng = np.random.default_rng(0)
    blocks = [(np.arange(n, dtype=np.int32), -1) for n in (3, 5, 1, 0, 2000, 40)] + [(np.arange(30, dtype=np.int32), 12)]
    units = make_units(blocks, True, batch_pairs=1000, shard_pairs=100_000)
    covered = {}
    for u in units:
        if u.shard is not None:
            k, refs, lo, hi = u.shard
            covered.setdefault(k, []).append((lo, hi))
        else:
            for k, _, _ in u.blocks:
                covered.setdefault(k, []).append(None)
    assert sorted(covered) == [0, 1, 4, 5, 6]  # empty and single-tuple partitions have no pairs
    shards = sorted(covered[4])
    assert len(shards) >= 2 and shards[0][0] == 0 and shards[-1][1] == 2000
    assert all(a[1] == b[0] for a, b in zip(shards, shards[1:]))
    total = sum(u.cost for u in units)
    assert total == sum(pair_count(len(r), s, True) for r, s in blocks)


def test_lpt_placement_and_stealing_visit_every_unit_once():
    costs = [random.Random(k).randint(1, 1000) for k in range(200)]
    units = [Unit(k, c) for k, c in enumerate(costs)]
    q = StealingQueues(units, 4)
    assert max(q.load) - min(q.load) <= max(costs)
    seen = []
    lock = threading.Lock()

    def device(d, delay):
        while True:
            u = q.next(d)
            if u is None:
                return
            time.sleep(delay * u.cost * 1e-6)
            with lock:
                seen.append(u.uid)

    ts = [threading.Thread(target=device, args=(d, 40 if d == 0 else 1)) for d in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert sorted(seen) == list(range(200))
    assert sum(q.steals[1:]) > 0  # the fast devices stole from the slow one


@pytest.mark.gpu
@pytest.mark.parametrize("devices,workers", [([0], 1), ([0], 2), ([0, 0, 0], 2)])
def test_multi_device_engine_matches_single_runs(devices, workers):
    rel, path, _ = goldens.load("citation")
    rng = random.Random(3)
    ids = list(range(len(rel)))
    rng.shuffle(ids)
    parts, k = [], 0
    while k < len(ids):
        size = rng.choice([2, 9, 40, 150, 900])
        parts.append(DataPartition(len(parts), tuple(ids[k:k + size])))
        k += size
    eng = MultiDeviceEngine(rel, path, devices=devices, workers_per_device=workers, batch_pairs=20_000,
                            shard_pairs=50_000)
    for cfg in (EngineConfig(), EngineConfig(symmetric_mode=False)):
        got = eng.run_partitions(parts, cfg)
        for p, cs in zip(parts, got):
            want = run_partition(p, rel, path, cfg)
            assert sorted(cs.pairs) == sorted(want.pairs)
            assert cs.stats.total_comparisons() == want.stats.total_comparisons()


@pytest.mark.gpu
def test_multi_device_engine_shards_one_big_partition():
    rel, path, cases = goldens.load("citation")
    eng = MultiDeviceEngine(rel, path, devices=[0, 0], workers_per_device=2, shard_pairs=1_000_000)
    cs = eng.run_partitions([DataPartition(0, tuple(range(len(rel))))])[0]
    assert sorted(cs.pairs) == goldens.expected_rows(cases[0])
    assert cs.stats.total_comparisons() == cases[0]["comparisons"]
    assert len(cs.stats.blocks) >= 8
