"""Host half of the boundary: exact threshold tables, program compilation,
encodings, plan construction and configuration -- all on the CPU."""

import math
import os
import random
import sys

import numpy as np
import pytest

from paper_2410_04349_b200 import EngineConfig, parse_ruleset, plan_from_stats, predicate_universe
from paper_2410_04349_b200.encode import (
    NEVER,
    OP_CHECKPOINT,
    RelationEncoding,
    compile_program,
    edit_tables,
    jaccard_tables,
)
from paper_2410_04349_b200.errors import ConfigError, RuleParseError
from paper_2410_04349_b200.text import fold_text, tokenize, value_text

import goldens

REF = "/root/reference/pkg/src"
HAVE_REF = os.path.isdir(REF)


# ---------------------------------------------------------------------------
# exact tables == the reference's float64 tests (encode.py:236-238, 256-259)


def _edit_ref(la, lb, lev, delta, prefilter=True):
    longest = max(la, lb)
    if longest == 0:
        return True
    if prefilter and longest - min(la, lb) > (1.0 - delta) * longest:
        return False
    return 1.0 - lev / longest >= delta


def _jac_ref(n, m, inter, delta, prefilter=True):
    if n == 0 and m == 0:
        return False
    small, big = min(n, m), max(n, m)
    if prefilter and small < delta * big:
        return False
    return inter / (n + m - inter) >= delta


DELTAS = [0.3, 0.34, 0.5, 0.55, 0.6, 0.7, 0.75, 0.8, 0.9, 0.97, 0.98, 1.0, 1 / 3, 2 / 3, 0.1, 0.01]


@pytest.mark.parametrize("delta", DELTAS)
@pytest.mark.parametrize("prefilter", [True, False])
def test_edit_tables_match_float_semantics(delta, prefilter):
    lmax = 130
    maxgap, maxd = edit_tables(delta, lmax, prefilter)
    rng = random.Random(int(delta * 1000) + prefilter)
    for _ in range(6000):
        la, lb = rng.randint(0, lmax), rng.randint(0, lmax)
        L = max(la, lb)
        lev = rng.randint(abs(la - lb), L) if L else 0
        want = _edit_ref(la, lb, lev, delta, prefilter)
        got = L == 0 or (abs(la - lb) <= maxgap[L] and lev <= maxd[L])
        assert got == want, (la, lb, lev, delta)


@pytest.mark.parametrize("delta", DELTAS)
@pytest.mark.parametrize("prefilter", [True, False])
def test_jaccard_tables_match_float_semantics(delta, prefilter):
    nmax = 60
    minsmall, mink = jaccard_tables(delta, nmax, prefilter)
    for n in range(nmax + 1):
        for m in range(nmax + 1):
            for inter in range(min(n, m) + 1):
                want = _jac_ref(n, m, inter, delta, prefilter)
                got = not (n == 0 and m == 0) and min(n, m) >= minsmall[max(n, m)] and inter >= mink[n + m]
                assert got == want, (n, m, inter, delta)


def test_survey_float_edges():
    # (1-0.3)*90 < 63 so the engine rejects a gap of 63 at L=90
    maxgap, maxd = edit_tables(0.3, 90, True)
    assert maxgap[90] == 62 and maxd[90] == 63
    minsmall, _ = jaccard_tables(0.55, 100, True)
    assert minsmall[100] == 56  # 0.55*100 = 55.00000000000001


def test_mink_never_when_unreachable():
    _, mink = jaccard_tables(1.0, 5, True)
    assert mink[3] == NEVER and mink[4] == 2


# ---------------------------------------------------------------------------
# program compilation


def test_program_arrays_follow_the_path():
    rel, path, _ = goldens.load("products")
    enc = RelationEncoding(rel).prepare(path.predicate_table)
    prog = compile_program(path, enc)
    assert len(prog.ins_op) == len(path.instructions)
    cps = [path.rule_ids[prog.ins_rule[k]] for k in range(len(prog.ins_op)) if prog.ins_op[k] == OP_CHECKPOINT]
    assert cps == path.checkpoint_order()
    for k, ins in enumerate(path.instructions):
        if hasattr(ins, "slot"):
            assert prog.ins_slot[k] == ins.slot and prog.ins_fail[k] == ins.fail_jump
    assert prog.n_slots == len(path.predicate_table) == 6


def test_program_limits_raise_config_error():
    doc = [{"id": f"r{k}", "when": [{"t_attr": "x", "op": "eq", "const": f"v{k}"}]} for k in range(70)]
    rules = parse_ruleset(__import__("json").dumps(doc))
    uni = predicate_universe(rules)
    path = plan_from_stats(rules, {p: 1.0 for p in uni}, {p: 0.5 for p in uni})
    from paper_2410_04349_b200.relation import relation_from_rows

    rel = relation_from_rows(["x"], ["short_text"], [["v1"], ["v2"]])
    with pytest.raises(ConfigError):
        compile_program(path, RelationEncoding(rel))


def test_unknown_measure_has_no_device_kernel():
    from paper_2410_04349_b200.relation import relation_from_rows
    from paper_2410_04349_b200.rules import Predicate

    rel = relation_from_rows(["x"], ["short_text"], [["a"], ["b"]])
    with pytest.raises(ConfigError):
        RelationEncoding(rel).slot_for(Predicate("x", "sim", "x", measure="cosine", threshold=0.5))
    with pytest.raises(RuleParseError):
        parse_ruleset('[{"id": "r", "when": [{"t_attr": "x", "op": "sim", "s_attr": "x", "measure": "cosine", '
                      '"threshold": 0.5}]}]')


def test_engine_config_validation():
    with pytest.raises(ConfigError):
        EngineConfig(n_t=0)
    with pytest.raises(ConfigError):
        EngineConfig(stealing="sometimes")
    with pytest.raises(ConfigError):
        EngineConfig(chunk_size=0)
    assert EngineConfig(symmetric_mode=False, enumerate_witnesses=True, device_stats=False).flags() == 2


def test_text_semantics():
    # pkg/tests/test_measures.py:101-102
    assert tokenize("15.6-inch (16GB) RAM") == ["156inch", "16gb", "ram"]
    assert fold_text("  MÜNCHEN ") == "münchen"
    assert value_text(12.0) == "12" and value_text(12.5) == "12.5"


# ---------------------------------------------------------------------------
# parity of the host layer with the reference itself (container only)


@pytest.mark.skipif(not HAVE_REF, reason="reference not importable here")
def test_plan_from_stats_equals_reference_plan():
    sys.path.insert(0, REF)
    sys.path.insert(0, os.path.join(os.path.dirname(REF), "tests"))
    from ruleblock.datasets import random_instance
    from ruleblock.planner.plan import build_tree, compile_path, order_predicates, score_tree
    from ruleblock.rules import parse_ruleset as ref_parse
    from ruleblock.rules import predicate_universe as ref_uni

    import json

    from paper_2410_04349_b200.plan import path_to_dict

    for seed in range(40):
        _, doc = random_instance(seed)
        rr = ref_parse(json.dumps(doc))
        uni = ref_uni(rr)
        rng = random.Random(seed)
        costs = {p: rng.choice([0.1, 0.3, 0.5, 1.0]) for p in uni}
        sps = {p: rng.choice([0.1, 0.2, 0.5, 0.8]) for p in uni}
        want = compile_path(score_tree(build_tree(rr, order_predicates(uni, costs, sps)), sps))
        ours_rules = parse_ruleset(json.dumps(doc))
        ocosts = {q: costs[p] for p, q in zip(uni, predicate_universe(ours_rules))}
        osps = {q: sps[p] for p, q in zip(uni, predicate_universe(ours_rules))}
        got = plan_from_stats(ours_rules, ocosts, osps)
        assert path_to_dict(got) == path_to_dict(want), seed


@pytest.mark.skipif(not HAVE_REF, reason="reference not importable here")
def test_encoding_accepts_reference_objects_and_matches_encoded_relation():
    sys.path.insert(0, REF)
    import tempfile

    from ruleblock.datasets import random_instance, rows_to_relation
    from ruleblock.encode import EncodedRelation

    with tempfile.TemporaryDirectory() as tmp:
        for seed in range(10):
            rows, _ = random_instance(seed)
            ref_rel = rows_to_relation(rows, ["cat", "num", "stext", "ltext"], tmp, name=f"e{seed}.csv")
            ref_enc = EncodedRelation(ref_rel)
            ours = RelationEncoding(ref_rel)  # duck-typed on the reference's Relation
            for attr in ("cat", "num", "stext"):
                a = ref_enc.eq_codes(attr)
                b = ours.columns[ours.get(("codes", attr))].data
                assert np.array_equal(a.astype(np.int64), b.astype(np.int64))
            for attr in ("stext", "ltext"):
                t = ref_enc.tokens(attr)
                c = ours.columns[ours.get(("tokens", attr))]
                assert np.array_equal(t.offsets, c.offsets) and np.array_equal(t.flat, c.data)
                ch = ref_enc.chars(attr)
                cc = ours.columns[ours.get(("chars", attr))]
                assert np.array_equal(ch.offsets, cc.offsets) and np.array_equal(ch.flat, cc.data)
                assert ch.flat.dtype == cc.data.dtype


class _Measure:
    def __init__(self, scorer, fold=True):
        self.scorer, self.fold = scorer, fold


class _Registry:
    def __init__(self, **entries):
        self.entries = entries

    def get(self, mid):
        if mid not in self.entries:
            raise ConfigError(f"unregistered measure {mid!r}")
        return self.entries[mid]


def _builtin(name):
    def f(a, b, fold=True):
        return 0.0
    f.__name__, f.__module__ = name, "ruleblock.measures"
    return f


def test_registry_scored_slots_refuse_custom_scorers():
    """The reference scores cross-attribute jaccard / exact_token and
    mixed-width edit through the registry (encode.py:281-324 ->
    measures.py:145-174): a custom scorer there raises ConfigError instead
    of being replaced by the built-in device measure."""
    rel, path, _ = goldens.load("edge_cross_attr")
    builtin = _Registry(edit=_Measure(_builtin("edit_score")), jaccard=_Measure(_builtin("jaccard_score")),
                        exact_token=_Measure(_builtin("exact_token_score")))
    enc = RelationEncoding(rel).prepare(path.predicate_table)
    compile_program(path, enc, builtin)  # built-in scorers: accepted
    for mid in ("jaccard", "exact_token"):
        custom = dict(builtin.entries)
        custom[mid] = _Measure(lambda a, b, fold=True: 1.0)
        with pytest.raises(ConfigError, match="custom scorer"):
            compile_program(path, RelationEncoding(rel).prepare(path.predicate_table), _Registry(**custom))
        custom[mid] = _Measure(_builtin(f"{mid}_score"), fold=False)
        with pytest.raises(ConfigError, match="custom scorer"):
            compile_program(path, RelationEncoding(rel).prepare(path.predicate_table), _Registry(**custom))
    # a same-attribute jaccard slot never consults the scorer (the reference's _jaccard_slot)
    rel2, path2, _ = goldens.load("products")
    custom = dict(builtin.entries, jaccard=_Measure(lambda a, b, fold=True: 1.0),
                  edit=_Measure(lambda a, b, fold=True: 1.0))
    compile_program(path2, RelationEncoding(rel2).prepare(path2.predicate_table), _Registry(**custom))


@pytest.mark.skipif(not HAVE_REF, reason="reference package not present")
def test_reference_default_registry_is_builtin():
    sys.path.insert(0, REF)
    from ruleblock.measures import Measure, default_registry

    rel, path, _ = goldens.load("edge_cross_attr")
    reg = default_registry()
    compile_program(path, RelationEncoding(rel).prepare(path.predicate_table), reg)
    reg.register(Measure("jaccard", lambda a, b, fold=True: 1.0))
    with pytest.raises(ConfigError):
        compile_program(path, RelationEncoding(rel).prepare(path.predicate_table), reg)
