"""Deferred verification (phase-1 survivors buffered, decided by a second
kernel): a range whose survivors overflow the buffer is rolled back and
re-run with room for all of them, and a range needing more than the buffer
limit is split until every piece fits (streaming).  Both paths are forced
with RB_SURV_MIN / RB_SURV_LIMIT and compared with the reference goldens."""

import pytest

import goldens


@pytest.fixture(autouse=True)
def _cold_programs(monkeypatch):
    """These tests drive the first-run streaming paths: programs must not
    start from the sizes an earlier program of the same shape learned."""
    monkeypatch.setenv("RB_LEARN", "0")
from paper_2410_04349_b200 import DataPartition, EngineConfig, run_cross, run_partition

CASES = ["citation", "products", "grouped", "edit_low", "skewed", "random_007", "random_031"]


def _replay(name):
    rel, path, cases = goldens.load(name)
    out = []
    for case in cases:
        cfg = EngineConfig(symmetric_mode=case["symmetric"], enumerate_witnesses=case["enumerate"])
        if case["left"] is not None:
            cs = run_cross(DataPartition(0, tuple(case["left"])), DataPartition(1, tuple(case["right"])), rel, path,
                           cfg)
        else:
            refs = tuple(range(len(rel))) if case["refs"] is None else tuple(case["refs"])
            cs = run_partition(DataPartition(0, refs), rel, path, cfg)
        assert sorted(cs.pairs) == goldens.expected_rows(case), (name, case["name"])
        assert cs.stats.total_comparisons() == case["comparisons"]
        out.append(cs)
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("name", [c for c in CASES if c in goldens.names()])
def test_survivor_buffer_overflow_reruns(name, monkeypatch):
    monkeypatch.delenv("RB_JIT", raising=False)
    monkeypatch.setenv("RB_SURV_MIN", "7")
    runs = _replay(name)
    surv = [cs.stats.blocks[0].survivors for cs in runs]
    assert any(s > 7 for s in surv)
    for cs, s in zip(runs, surv):
        if s > 7:  # ref check, then the first pair launch overflowed and was rolled back: pair, pair + verify
            assert cs.stats.launches == 4


@pytest.mark.gpu
@pytest.mark.parametrize("name", [c for c in CASES if c in goldens.names()])
def test_survivor_limit_streams_in_ranges(name, monkeypatch):
    monkeypatch.delenv("RB_JIT", raising=False)
    monkeypatch.setenv("RB_SURV_MIN", "3")
    monkeypatch.setenv("RB_SURV_LIMIT", "5")
    runs = _replay(name)
    for cs in runs:
        assert cs.stats.specialized
        if cs.stats.blocks[0].survivors > 5:
            assert cs.stats.launches > 3


@pytest.mark.gpu
@pytest.mark.parametrize("flavour", ["specialized", "generic"])
def test_out_of_range_ref_fails_loudly(flavour, monkeypatch):
    """A tuple ref outside the relation is caught on the device before any
    pair is evaluated, and reported with its position."""
    from paper_2410_04349_b200.errors import ConfigError

    if flavour == "generic":
        monkeypatch.setenv("RB_JIT", "0")
    else:
        monkeypatch.delenv("RB_JIT", raising=False)
    rel, path, _ = goldens.load("products")
    with pytest.raises(ConfigError, match="position 3"):
        run_partition(DataPartition(0, (0, 1, 2, len(rel) + 7)), rel, path)
    with pytest.raises(ConfigError, match="outside the relation"):
        run_cross(DataPartition(0, (0, 1)), DataPartition(1, (len(rel),)), rel, path)


@pytest.mark.gpu
@pytest.mark.parametrize("name", [c for c in CASES if c in goldens.names()])
def test_output_grows_in_place_across_ranges(name, monkeypatch):
    """Tiny survivor budget (many ranges) and a 2-row initial output buffer:
    rows already written must survive every in-place growth."""
    monkeypatch.delenv("RB_JIT", raising=False)
    monkeypatch.setenv("RB_SURV_MIN", "2")
    monkeypatch.setenv("RB_SURV_LIMIT", "16")
    monkeypatch.setenv("RB_OUT_MIN", "2")
    _replay(name)


@pytest.mark.gpu
def test_batched_output_growth_keeps_parts(monkeypatch):
    """The same with a batched run: the partition index of every kept row
    must move with it."""
    from paper_2410_04349_b200 import run_partitions

    monkeypatch.delenv("RB_JIT", raising=False)
    rel, path, cases = goldens.load("citation")
    parts = [DataPartition(k, tuple(range(k * 400, min(len(rel), k * 400 + 700)))) for k in range(10)]
    want = [run_partition(p, rel, path).sorted_pairs() for p in parts]
    monkeypatch.setenv("RB_SURV_MIN", "2")
    monkeypatch.setenv("RB_SURV_LIMIT", "64")
    monkeypatch.setenv("RB_OUT_MIN", "2")
    got = [cs.sorted_pairs() for cs in run_partitions(parts, rel, path)]
    assert got == want and sum(map(len, want)) > 10


@pytest.mark.gpu
def test_useless_gate_switches_off_and_stays_exact(monkeypatch):
    """Stage-1 equality key that every pair passes (a constant column): after
    the first run the program switches to its ungated variant; every run must
    match the oracle."""
    import json
    import random

    from paper_2410_04349_b200 import EngineConfig
    from paper_2410_04349_b200.engine import PathProgram, _encoding_for
    from paper_2410_04349_b200.plan import plan_from_stats
    from paper_2410_04349_b200.relation import relation_from_rows
    from paper_2410_04349_b200.rules import parse_ruleset, predicate_universe

    monkeypatch.delenv("RB_JIT", raising=False)
    monkeypatch.delenv("RB_GATE", raising=False)
    rng = random.Random(3)
    words = ["alpha", "beta", "gamma", "delta", "eps", "zeta", "eta", "theta"]
    rows = [["k", " ".join(rng.choices(words, k=rng.randint(2, 6))), "".join(rng.choices("abc", k=rng.randint(3, 9))),
             f"z{rng.randrange(3)}"] for _ in range(900)]
    rel = relation_from_rows(["blk", "title", "name", "zip"], ["short_text", "long_text", "short_text", "short_text"],
                             rows)
    rules = parse_ruleset(json.dumps([
        {"id": "A", "when": [{"t_attr": "blk", "op": "eq", "s_attr": "blk"},
                             {"t_attr": "title", "op": "sim", "s_attr": "title", "measure": "jaccard",
                              "threshold": 0.6}]},
        {"id": "B", "when": [{"t_attr": "blk", "op": "eq", "s_attr": "blk"},
                             {"t_attr": "zip", "op": "eq", "s_attr": "zip"},
                             {"t_attr": "name", "op": "sim", "s_attr": "name", "measure": "edit", "threshold": 0.7}]}]))
    uni = predicate_universe(rules)
    path = plan_from_stats(rules, {p: (0.1 if p.comparator == "eq" else 1.0) for p in uni}, {p: 0.5 for p in uni})
    enc = _encoding_for(rel, None)
    enc.prepare(path.predicate_table)
    prog = PathProgram(path, enc)
    case = {"symmetric": True, "enumerate": False, "refs": None, "left": None, "right": None}
    want, cmp = goldens.oracle_rows(rel, path, case)
    for _ in range(3):
        cs = run_partition(DataPartition(0, tuple(range(len(rel)))), rel, path, EngineConfig(), program=prog)
        assert sorted(cs.pairs) == want and cs.stats.total_comparisons() == cmp
    assert len(want) > 0


@pytest.mark.gpu
@pytest.mark.parametrize("symmetric", [True, False])
@pytest.mark.parametrize("sizes", ["mixed", "tiny", "tiny_enumerate"])
def test_many_part_batch_items_built_by_threads(symmetric, sizes, monkeypatch):
    """A batch of many partitions has its work items laid out by several
    host threads (forced here for any size with RB_ITEM_THREADS_MIN=1), and a
    batch of tiny symmetric partitions runs packed (several partitions per
    item; RB_PACK_MAX=0 turns packing off): the rows of every partition
    equal its own single run."""
    import random

    from paper_2410_04349_b200 import run_partitions

    monkeypatch.delenv("RB_JIT", raising=False)
    monkeypatch.delenv("RB_PACK_MAX", raising=False)
    rel, path, _ = goldens.load("citation")
    rng = random.Random(7)
    parts, k = [], 0
    choice = [1, 2, 3, 5, 9, 17, 40, 130, 700, 1300] if sizes == "mixed" else [1, 2, 3, 5, 9, 17, 33, 64, 65, 90]
    while len(parts) < 300:
        size = rng.choice(choice)
        refs = rng.sample(range(len(rel)), size)
        parts.append(DataPartition(k, tuple(refs)))
        k += 1
    cfg = EngineConfig(symmetric_mode=symmetric, enumerate_witnesses=sizes.endswith("enumerate"))
    want = [run_partition(p, rel, path, cfg).sorted_pairs() for p in parts]
    for threads_min, pack in (("1", "64"), ("1000000", "64"), ("1", "0"), ("1", "100"), ("1", "100000")):
        monkeypatch.setenv("RB_ITEM_THREADS_MIN", threads_min)
        monkeypatch.setenv("RB_PACK_MAX", pack)
        got = [cs.sorted_pairs() for cs in run_partitions(parts, rel, path, cfg)]
        assert got == want, (threads_min, pack)
        assert [cs.stats.total_comparisons() for cs in run_partitions(parts, rel, path, cfg)] == \
               [len(p.tuple_refs) * (len(p.tuple_refs) - 1) // (2 if symmetric else 1) for p in parts]
    assert sum(map(len, want)) > 50


@pytest.mark.gpu
def test_repeated_run_replays_the_ranges_that_fit(monkeypatch):
    """A program run again over the same items replays the previous run's
    survivor ranges: no overflow re-runs the second time, same rows."""
    import numpy as np

    from paper_2410_04349_b200._lib import RB_SYMMETRIC
    from paper_2410_04349_b200.encode import RelationEncoding
    from paper_2410_04349_b200.engine import PathProgram

    monkeypatch.delenv("RB_JIT", raising=False)
    monkeypatch.setenv("RB_SURV_MIN", "2")
    monkeypatch.setenv("RB_SURV_LIMIT", "64")
    rel, path, _ = goldens.load("citation")
    enc = RelationEncoding(rel).prepare(path.predicate_table)
    prog = PathProgram(path, enc, device=0)
    (t1, s1, r1), st1 = prog.run_raw(None, len(rel), RB_SYMMETRIC)
    (t2, s2, r2), st2 = prog.run_raw(None, len(rel), RB_SYMMETRIC)
    rows1 = sorted(zip(t1.tolist(), s1.tolist(), r1.tolist()))
    assert rows1 == sorted(zip(t2.tolist(), s2.tolist(), r2.tolist())) and len(rows1) > 100
    assert st1.retries > 0 and st2.retries == 0 and st2.launches < st1.launches
    assert st1.comparisons == st2.comparisons == len(rel) * (len(rel) - 1) // 2


@pytest.mark.gpu
def test_optimistic_range_overflow_rolls_back(monkeypatch):
    """A range queued optimistically (pair + verify with one host wait, on the
    survivor rate of the program's previous run) that overflows the survivor
    buffer is rolled back and re-run through the checked path: same rows as a
    fresh program, at least one retry."""
    import numpy as np

    from paper_2410_04349_b200._lib import RB_SYMMETRIC
    from paper_2410_04349_b200.encode import RelationEncoding
    from paper_2410_04349_b200.engine import PathProgram

    monkeypatch.delenv("RB_JIT", raising=False)
    rel, path, _ = goldens.load("citation")
    enc = RelationEncoding(rel).prepare(path.predicate_table)
    fresh = PathProgram(path, enc, device=0)
    (t0, s0, r0), st0 = fresh.run_raw(None, len(rel), RB_SYMMETRIC)
    want = sorted(zip(t0.tolist(), s0.tolist(), r0.tolist()))
    assert st0.survivors > 8 and len(want) > 100

    monkeypatch.setenv("RB_SURV_MIN", "8")
    monkeypatch.setenv("RB_SURV_LIMIT", "8")  # the range sizing cannot grow the buffer ahead
    monkeypatch.setenv("RB_OPT_MARGIN", "0")
    prog = PathProgram(path, enc, device=0)
    # a run without survivors teaches the program a zero survivor rate ...
    for k in range(1, len(rel)):
        _, st1 = prog.run_raw(np.array([0, k], dtype=np.int32), 2, RB_SYMMETRIC)
        if st1.survivors == 0:
            break
    assert st1.survivors == 0
    # ... so the whole relation's first range is queued optimistically and overflows
    (t2, s2, r2), st2 = prog.run_raw(None, len(rel), RB_SYMMETRIC)
    assert sorted(zip(t2.tolist(), s2.tolist(), r2.tolist())) == want
    assert st2.retries >= 1 and st2.comparisons == st0.comparisons
