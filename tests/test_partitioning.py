"""Plan-derived partitioning restated in pipeline.py must
produce the reference's partitions exactly: same pids, refs, branches, key
groups and sibling groups (reference importable in the build container)."""

import json
import os
import sys
import tempfile

import numpy as np
import pytest

from paper_2410_04349_b200.pipeline import BandingConfig, collect, iter_partitions, mix64, sibling_pull_pairs, stable_hash64

REF = "/root/reference/pkg/src"
HAVE_REF = os.path.isdir(REF)


def test_hash_helpers_are_deterministic():
    assert stable_hash64("abc", 0) == stable_hash64("abc", 0) != stable_hash64("abc", 1)
    x = np.array([1, 2, 3], dtype=np.uint64)
    assert np.array_equal(mix64(x, 5), mix64(x, 5))


@pytest.mark.skipif(not HAVE_REF, reason="reference not importable here")
@pytest.mark.parametrize("max_size", [3, 16, 512])
def test_partitions_equal_reference(max_size):
    sys.path.insert(0, REF)
    from ruleblock.bench import FAST_PLANNER
    from ruleblock.datasets import CITATION_HEADER, citation_benchmark, random_instance, rows_to_relation
    from ruleblock.partitioning import BandingConfig as RB
    from ruleblock.partitioning import derive_partitioners
    from ruleblock.partitioning import iter_partitions as ref_iter
    from ruleblock.partitioning import sibling_pull_pairs as ref_pulls
    from ruleblock.planner.plan import generate_plan
    from ruleblock.rules import parse_ruleset

    with tempfile.TemporaryDirectory() as tmp:
        cases = []
        for seed in range(6):
            rows, doc = random_instance(seed)
            cases.append((rows_to_relation(rows, ["cat", "num", "stext", "ltext"], tmp, name=f"p{seed}.csv"), doc))
        rows, doc, _ = citation_benchmark(n_tuples=800, n_matches=300)
        cases.append((rows_to_relation(rows, CITATION_HEADER, tmp, name="cit.csv"), doc))
        for rel, doc in cases:
            bundle = generate_plan(rel, parse_ruleset(json.dumps(doc)), FAST_PLANNER)
            want = list(ref_iter(rel, derive_partitioners(bundle.tree, RB(rows=4, seed=0)), max_size))
            got = list(iter_partitions(rel, bundle.path, max_size, BandingConfig(rows=4, seed=0)))
            assert [(p.pid, p.tuple_refs, p.branch_id, p.key_group, p.sibling_group) for p in got] == \
                   [(p.pid, p.tuple_refs, p.branch_id, p.key_group, p.sibling_group) for p in want]
            assert sibling_pull_pairs(got) == ref_pulls(want)


def test_collect_keeps_earliest_rule_per_pair():
    from paper_2410_04349_b200.engine import CandidateSet

    a = CandidateSet(arrays=(np.array([1, 1, 2]), np.array([5, 5, 3]), np.array([2, 0, 1])), rule_ids=["a", "b", "c"])
    b = CandidateSet(arrays=(np.array([1, 4]), np.array([5, 7]), np.array([1, 2])), rule_ids=["a", "b", "c"])
    cs = collect([a, b], ["a", "b", "c"])
    assert sorted(cs.pairs) == [(1, 5, "a"), (2, 3, "b"), (4, 7, "c")]


@pytest.mark.parametrize("max_size", [2, 5, 64])
def test_plan_partitions_equal_pipeline(max_size):
    """synth.plan_partitions (the config 4 (i) bench blocks, from encoded code
    columns) yields exactly pipeline_run's partitions and sibling pulls."""
    import random

    from paper_2410_04349_b200.encode import RelationEncoding
    from paper_2410_04349_b200.plan import plan_from_stats
    from paper_2410_04349_b200.relation import MISSING, relation_from_rows
    from paper_2410_04349_b200.rules import parse_ruleset, predicate_universe
    from paper_2410_04349_b200.synth import plan_partitions

    rng = random.Random(max_size)
    rows = [[rng.choice(["x", " x", "y", "z ", MISSING]), float(rng.randint(0, 3)), rng.choice(["ab", "abc", "b"])]
            for _ in range(120)]
    rel = relation_from_rows(["k", "n", "s"], ["short_text", "numeric", "short_text"], rows)
    doc = [{"id": "a", "when": [{"t_attr": "k", "op": "eq", "s_attr": "k"},
                               {"t_attr": "s", "op": "sim", "s_attr": "s", "measure": "edit", "threshold": 0.6}]},
           {"id": "b", "when": [{"t_attr": "n", "op": "eq", "s_attr": "n"}]}]
    rules = parse_ruleset(json.dumps(doc))
    uni = predicate_universe(rules)
    path = plan_from_stats(rules, {p: 1.0 for p in uni}, {p: 0.5 for p in uni})
    enc = RelationEncoding(rel).prepare(path.predicate_table)
    parts = list(iter_partitions(rel, path, max_size))
    by = {p.pid: p for p in parts}
    want = [(tuple(p.tuple_refs), -1) for p in parts if len(p.tuple_refs) > 1]
    want += [(tuple(by[a].tuple_refs) + tuple(by[b].tuple_refs), len(by[a].tuple_refs))
             for a, b in sibling_pull_pairs(parts)]
    got = [(tuple(int(x) for x in r), int(sp)) for r, sp in plan_partitions(enc, path, max_size)]
    assert sorted(got) == sorted(want)
    assert any(sp >= 0 for _, sp in got) == (max_size < 40)


def test_eq_branch_keys_from_codes_equal_key_strings():
    """pipeline.eq_branch_keys (key strings formed once per distinct value,
    from the encoding's codes) == rank_keys(branch_keys(...)) (the
    reference's key string of every tuple) on every equality root of the
    fixtures."""
    import numpy as np

    from paper_2410_04349_b200.encode import RelationEncoding
    from paper_2410_04349_b200.pipeline import (BandingConfig, branch_keys, branch_order, eq_branch_keys, rank_keys,
                                                root_predicates)

    import goldens

    checked = 0
    for name in goldens.pipeline_names() + goldens.names():
        rel, path, _ = goldens.load(name)
        enc = RelationEncoding(rel)
        for b in branch_order(path):
            pred = root_predicates(path)[b]
            if pred.comparator != "eq" or pred.is_cross_attr or pred.rhs_attr is None:
                continue
            got = eq_branch_keys(rel, enc, pred)
            want = rank_keys(branch_keys(rel, pred, BandingConfig()))
            assert np.array_equal(got[0], want[0]) and got[1] == want[1], (name, b)
            checked += 1
    assert checked > 30
