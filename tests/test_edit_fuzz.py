"""Bounded edit distance on the device (Landau-Vishkin for maxd <= 31, the
banded DP above) against the CPU oracle's full two-row DP: near-duplicate
strings of 0-120 characters, ASCII and non-ASCII columns, missing and blank
cells, thresholds whose maxd[L] spans 0..60."""

import json
import random

import pytest

import goldens
from paper_2410_04349_b200 import DataPartition, EngineConfig, run_partition
from paper_2410_04349_b200.plan import plan_from_stats
from paper_2410_04349_b200.relation import MISSING, relation_from_rows
from paper_2410_04349_b200.rules import parse_ruleset, predicate_universe


def _perturb(rng, s, k, alpha):
    b = list(s)
    for _ in range(k):
        op = rng.randrange(3)
        p = rng.randrange(len(b) + 1)
        if op == 0 and p < len(b):
            b[p] = rng.choice(alpha)
        elif op == 1:
            b.insert(p, rng.choice(alpha))
        elif b and p < len(b):
            del b[p]
    return "".join(b)


def make(seed, n=160, unicode=False):
    rng = random.Random(seed)
    alpha = "abcd" if seed % 2 else "abcdefghij klmnop"
    if unicode:
        alpha += "éßΩж"
    rows = []
    while len(rows) < n:
        base = "".join(rng.choice(alpha) for _ in range(rng.randint(0, 120)))
        for _ in range(rng.randint(1, 8)):
            x = rng.random()
            if x < 0.05:
                rows.append([MISSING])
            elif x < 0.08:
                rows.append(["" if rng.random() < 0.5 else "   "])
            else:
                rows.append([_perturb(rng, base, rng.randint(0, 12), alpha)])
    rows = rows[:n]
    rel = relation_from_rows(["s"], ["long_text"], rows)
    doc = [{"id": f"e{k}", "when": [{"t_attr": "s", "op": "sim", "s_attr": "s", "measure": "edit", "threshold": th}]}
           for k, th in enumerate(rng.sample([0.3, 0.5, 0.7, 0.8, 0.9, 0.95, 0.98], 3))]
    rules = parse_ruleset(json.dumps(doc))
    uni = predicate_universe(rules)
    path = plan_from_stats(rules, {p: 1.0 for p in uni}, {p: 0.5 for p in uni})
    return rel, path


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(10))
@pytest.mark.parametrize("unicode", [False, True])
@pytest.mark.parametrize("fold", ["auto", "1"])
def test_edit_distance_gpu_vs_oracle(seed, unicode, fold, monkeypatch):
    """fold=1 forces the 8-bucket (folded) bag filter on every string feature."""
    if fold == "auto":
        monkeypatch.delenv("RB_FOLD_BAG", raising=False)
    else:
        monkeypatch.setenv("RB_FOLD_BAG", fold)
    rel, path = make(seed, unicode=unicode)
    refs = list(range(len(rel)))
    random.Random(seed).shuffle(refs)
    for sym, enum in ((True, True), (False, False)):
        cfg = EngineConfig(symmetric_mode=sym, enumerate_witnesses=enum)
        cs = run_partition(DataPartition(0, tuple(refs)), rel, path, cfg)
        case = {"symmetric": sym, "enumerate": enum, "refs": refs, "left": None, "right": None}
        want, cmp = goldens.oracle_rows(rel, path, case)
        assert sorted(cs.pairs) == want
        assert cs.stats.total_comparisons() == cmp


def test_fuzz_relation_has_matches():
    rel, path = make(0)
    case = {"symmetric": True, "enumerate": True, "refs": None, "left": None, "right": None}
    want, _ = goldens.oracle_rows(rel, path, case)
    assert len(want) > 50


def make_long(seed, n=70):
    """Long strings with low thresholds: maxd[L] far above 31, so the
    device runs Myers' bit-vector algorithm (and its fallbacks: patterns
    over 1024 characters or with more than 48 distinct characters)."""
    rng = random.Random(seed)
    alpha = ["abcdefghij ", "abcdefghijklmnopqrstuvwxyz ", "abcdefghijklmnopqrstuvwxyzABCDEFGHIJKLMNOPQRSTUVWXYZ0123456789",
             "abcdeéßΩжйк "][seed % 4]
    rows = []
    while len(rows) < n:
        L = rng.choice([40, 150, 300, 700, 1100]) + rng.randint(0, 40)
        base = "".join(rng.choice(alpha) for _ in range(L))
        for _ in range(rng.randint(1, 6)):
            rows.append([_perturb(rng, base, rng.choice([0, 3, 30, 120, 400]), alpha)])
    rel = relation_from_rows(["s"], ["long_text"], rows[:n])
    doc = [{"id": f"e{k}", "when": [{"t_attr": "s", "op": "sim", "s_attr": "s", "measure": "edit", "threshold": th}]}
           for k, th in enumerate(rng.sample([0.3, 0.45, 0.55, 0.7, 0.8, 0.9], 3))]
    rules = parse_ruleset(json.dumps(doc))
    uni = predicate_universe(rules)
    return rel, plan_from_stats(rules, {p: 1.0 for p in uni}, {p: 0.5 for p in uni})


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(8))
def test_long_strings_large_bounds_gpu_vs_oracle(seed):
    rel, path = make_long(seed)
    refs = list(range(len(rel)))
    for sym in (True, False):
        cfg = EngineConfig(symmetric_mode=sym, enumerate_witnesses=True)
        cs = run_partition(DataPartition(0, tuple(refs)), rel, path, cfg)
        case = {"symmetric": sym, "enumerate": True, "refs": None, "left": None, "right": None}
        want, cmp = goldens.oracle_rows(rel, path, case)
        assert sorted(cs.pairs) == want
        assert cs.stats.total_comparisons() == cmp


def test_long_fuzz_has_large_bounds_and_matches():
    from paper_2410_04349_b200.encode import RelationEncoding, compile_program

    for seed in range(4):
        rel, path = make_long(seed)
        case = {"symmetric": True, "enumerate": True, "refs": None, "left": None, "right": None}
        want, _ = goldens.oracle_rows(rel, path, case)
        assert len(want) > 0
        enc = RelationEncoding(rel).prepare(path.predicate_table)
        prog = compile_program(path, enc)
        assert prog.tables.max() > 300  # some maxd[L] far above the diagonal algorithm's 31
