"""Randomised program shapes: GPU (both kernels) vs the CPU oracle."""

import random

import numpy as np
import pytest

import goldens
import randwork
from paper_2410_04349_b200 import DataPartition, EngineConfig, run_cross, run_partition


def _oracle(rel, path, refs, split, flags):
    case = {"symmetric": bool(flags & 1), "enumerate": bool(flags & 2),
            "refs": None if split >= 0 else list(refs), "left": list(refs[:split]) if split >= 0 else None,
            "right": list(refs[split:]) if split >= 0 else None}
    return goldens.oracle_rows(rel, path, case)


def test_generator_shapes():
    shapes = [len(randwork.make(s)[2].predicate_table) for s in range(12)]
    assert max(shapes) > 10


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(24))
@pytest.mark.parametrize("flavour", ["specialized", "generic", "plain"])
def test_random_shapes_gpu_vs_oracle(seed, flavour, monkeypatch):
    """specialized: the default kernel (composite keys, implied kills, stage-1
    gate); generic: the statically built kernel; plain: specialised without
    composite keys and without the gate."""
    monkeypatch.delenv("RB_JIT", raising=False)
    monkeypatch.delenv("RB_GATE", raising=False)
    monkeypatch.delenv("RB_COMPOSITE", raising=False)
    if flavour == "generic":
        monkeypatch.setenv("RB_JIT", "0")
    elif flavour == "plain":
        monkeypatch.setenv("RB_GATE", "0")
        monkeypatch.setenv("RB_COMPOSITE", "0")
    rel, rules, path = randwork.make(seed)
    rng = random.Random(seed)
    n = len(rel)
    refs = list(range(n))
    rng.shuffle(refs)
    for sym, enum in ((True, False), (False, False), (True, True)):
        cfg = EngineConfig(symmetric_mode=sym, enumerate_witnesses=enum)
        flags = (1 if sym else 0) | (2 if enum else 0)
        cs = run_partition(DataPartition(0, tuple(refs)), rel, path, cfg)
        want, cmp = _oracle(rel, path, refs, -1, flags)
        assert sorted(cs.pairs) == want
        assert cs.stats.total_comparisons() == cmp
    half = n // 3
    cs = run_cross(DataPartition(0, tuple(refs[:half])), DataPartition(1, tuple(refs[half:])), rel, path)
    want, cmp = _oracle(rel, path, refs, half, 1)
    assert sorted(cs.pairs) == want and cs.stats.total_comparisons() == cmp
