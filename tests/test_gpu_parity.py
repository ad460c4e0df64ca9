"""CUDA path vs the reference's golden vectors and vs the CPU oracle.

Every case runs through the drop-in API (run_partition / run_cross), i.e.
through librbgpu.so's C ABI on cuda:0, and must match bit-exactly: the same
sorted (t, s, rule_id) rows and the same comparison count."""

import numpy as np
import pytest

import goldens
from paper_2410_04349_b200 import DataPartition, EngineConfig, run_cross, run_partition
from paper_2410_04349_b200.engine import PathProgram

pytestmark = pytest.mark.gpu

NAMES = goldens.names()


def gpu_rows(rel, path, case, prog=None):
    cfg = EngineConfig(symmetric_mode=case["symmetric"], enumerate_witnesses=case["enumerate"])
    if case["left"] is not None:
        cs = run_cross(DataPartition(-2, tuple(case["left"])), DataPartition(-3, tuple(case["right"])), rel, path,
                       cfg, program=prog)
    else:
        refs = tuple(range(len(rel))) if case["refs"] is None else tuple(case["refs"])
        cs = run_partition(DataPartition(0, refs), rel, path, cfg, program=prog)
    return sorted(cs.pairs), cs


@pytest.fixture(params=["specialized", "generic", "sig64", "sig128"])
def kernel_flavour(request, monkeypatch):
    """Run every case through the NVRTC-specialised kernel, the generic
    (statically built) kernel, and with the token signature forced to the
    folded 64-bit and the full 128-bit form."""
    monkeypatch.delenv("RB_JIT", raising=False)
    monkeypatch.delenv("RB_SIG64", raising=False)
    if request.param == "generic":
        monkeypatch.setenv("RB_JIT", "0")
    elif request.param == "sig64":
        monkeypatch.setenv("RB_SIG64", "1")
    elif request.param == "sig128":
        monkeypatch.setenv("RB_SIG64", "0")
    return request.param


@pytest.mark.parametrize("name", NAMES)
def test_gpu_matches_reference_golden(name, kernel_flavour):
    rel, path, cases = goldens.load(name)
    for case in cases:
        got, cs = gpu_rows(rel, path, case)
        assert got == goldens.expected_rows(case), f"{name}/{case['name']}"
        assert cs.stats.total_comparisons() == case["comparisons"], f"{name}/{case['name']}"
        evals = cs.stats.blocks[0].slot_evals
        assert (evals <= cs.stats.total_comparisons()).all()
        assert cs.stats.specialized == (kernel_flavour != "generic"), cs.stats.jit_log


def test_empty_and_singleton_partitions():
    rel, path, _ = goldens.load("products")
    assert len(run_partition(None, rel, path)) == 0
    cs = run_partition(DataPartition(0, (3,)), rel, path)
    assert len(cs) == 0 and cs.stats.total_comparisons() == 0


def test_program_reuse_across_partitions():
    rel, path, cases = goldens.load("random_001")
    from paper_2410_04349_b200.encode import RelationEncoding

    enc = RelationEncoding(rel).prepare(path.predicate_table)
    prog = PathProgram(path, enc)
    for case in cases:
        got, _ = gpu_rows(rel, path, case, prog=prog)
        assert got == goldens.expected_rows(case)


@pytest.mark.parametrize("name", ["citation", "random_052", "grouped"])
def test_row_shards_union_equals_whole(name):
    """rb_run_partition_rows over an equal-pair split == run_partition."""
    from paper_2410_04349_b200 import run_partition_rows, split_rows_by_pairs

    rel, path, cases = goldens.load(name)
    case = cases[0]
    part = DataPartition(0, tuple(range(len(rel))))
    got, cmp = [], 0
    for lo, hi in split_rows_by_pairs(len(rel), 3):
        cs = run_partition_rows(part, rel, path, lo, hi)
        got += cs.pairs
        cmp += cs.stats.total_comparisons()
    assert sorted(got) == goldens.expected_rows(case)
    assert cmp == case["comparisons"]



def test_batched_partitions_equal_single_runs():
    """run_partitions (one launch) == run_partition per partition, on a
    mix of shuffled / tiny / empty partitions and every golden relation."""
    import random

    from paper_2410_04349_b200 import run_partitions

    for name in ["random_052", "random_001", "citation", "edge_cross_attr", "products"]:
        rel, path, cases = goldens.load(name)
        rng = random.Random(7)
        ids = list(range(len(rel)))
        rng.shuffle(ids)
        parts, k = [], 0
        while k < len(ids):
            size = rng.choice([1, 2, 3, 17, 60, 300, 700])
            parts.append(DataPartition(len(parts), tuple(ids[k:k + size])))
            k += size
        parts.append(None)
        for sym in (True, False):
            cfg = EngineConfig(symmetric_mode=sym)
            batched = run_partitions(parts, rel, path, cfg)
            for p, cs in zip(parts, batched):
                single = run_partition(p, rel, path, cfg)
                assert sorted(cs.pairs) == sorted(single.pairs), name
                assert cs.stats.total_comparisons() == single.stats.total_comparisons()


def test_batched_crosses_equal_single_runs():
    from paper_2410_04349_b200 import run_crosses

    rel, path, _ = goldens.load("random_053")
    n = len(rel)
    pairs = [(DataPartition(0, tuple(range(0, k))), DataPartition(1, tuple(range(k, min(n, 2 * k + 5)))))
             for k in (1, 5, 20, n // 3)]
    batched = run_crosses(pairs, rel, path)
    for (l, r), cs in zip(pairs, batched):
        single = run_cross(l, r, rel, path)
        assert sorted(cs.pairs) == sorted(single.pairs)
        assert cs.stats.total_comparisons() == len(l) * len(r)


def test_evaluate_pair_known_answers():
    """pkg/tests/test_engine.py:68-118 on the device."""
    from paper_2410_04349_b200 import PairBitmaps, evaluate_pair

    rel, path, _ = goldens.load("products")
    T = rel.tuples
    bm = PairBitmaps.for_path(path)
    assert evaluate_pair(path, T[0], T[3], bm, None, rel.schema) == "phi1"
    bm.reset()
    assert evaluate_pair(path, T[1], T[2], bm, None, rel.schema) == "phi2"
    bm.reset()
    assert evaluate_pair(path, T[1], T[2], bm, None, rel.schema, all_witnesses=True) == ["phi2", "phi3"]
    bm.reset()
    evaluate_pair(path, T[0], T[4], bm, None, rel.schema)
    assert bm.scorer_calls.max() <= 1


@pytest.mark.gpu
@pytest.mark.parametrize("name", [n for n in goldens.names() if n.startswith(("random_0", "products", "edge", "grouped"))][:40])
def test_exact_slot_evals_equal_oracle_first_touch(name):
    """RB_EXACT_STATS: the device's per-slot first-touch counts over every
    pair equal the oracle's (evaluate_pair semantics, engine.py:122-128;
    SURVEY 8d E_s) -- for partitions, shuffled refs and cross runs."""
    from oracle import oracle
    from paper_2410_04349_b200.encode import RelationEncoding, compile_program

    rel, path, cases = goldens.load(name)
    enc = RelationEncoding(rel).prepare(path.predicate_table)
    prog = compile_program(path, enc)
    for case in cases:
        cfg = EngineConfig(symmetric_mode=case["symmetric"], enumerate_witnesses=case["enumerate"],
                           exact_slot_evals=True)
        flags = (1 if case["symmetric"] else 0) | (2 if case["enumerate"] else 0)
        if case["left"] is not None:
            left, right = DataPartition(0, tuple(case["left"])), DataPartition(1, tuple(case["right"]))
            cs = run_cross(left, right, rel, path, cfg)
            refs = np.array(case["left"] + case["right"], dtype=np.int32)
            _, cmp, ev = oracle.run(enc, prog, refs, len(refs), split=len(case["left"]), flags=flags)
        else:
            refs = tuple(range(len(rel))) if case["refs"] is None else tuple(case["refs"])
            cs = run_partition(DataPartition(0, refs), rel, path, cfg)
            _, cmp, ev = oracle.run(enc, prog, np.array(refs, dtype=np.int32), len(refs), flags=flags)
        got = np.sum([b.slot_evals for b in cs.stats.blocks], axis=0)
        assert cs.stats.total_comparisons() == cmp
        assert got.tolist() == np.asarray(ev).tolist(), (name, case["name"])


@pytest.mark.parametrize("name", ["products", "edge_direction", "edge_cross_attr", "random_007", "random_031",
                                  "random_064", "grouped"])
def test_evaluate_pairs_batch_equals_oracle_witness(name):
    """evaluate_pairs: many ordered pairs in one launch, each == the
    oracle's first witness evaluated t-then-s (evaluate_pair semantics)."""
    from oracle import oracle
    from paper_2410_04349_b200 import evaluate_pairs
    from paper_2410_04349_b200.encode import RelationEncoding, compile_program

    rel, path, _ = goldens.load(name)
    n = len(rel)
    rng = np.random.default_rng(3)
    pairs = rng.integers(0, n, size=(min(4000, n * n), 2)).astype(np.int32)
    pairs = pairs[pairs[:, 0] != pairs[:, 1]]
    got = evaluate_pairs(path, rel, pairs)
    enc = RelationEncoding(rel).prepare(path.predicate_table)
    prog = compile_program(path, enc)
    want = oracle.witness(enc, prog, pairs[:, 0], pairs[:, 1])
    assert got == [None if w < 0 else path.rule_ids[w] for w in want.tolist()]


@pytest.mark.parametrize("symmetric", [True, False])
@pytest.mark.parametrize("mixed", ["1", "0"])
def test_mixed_size_batch_runs_in_two_classes(symmetric, mixed, monkeypatch):
    """A batch of large (>= 768-tuple) and tiny units runs as two size
    classes (rb::run_mixed): every unit's rows -- recovered through the
    merged result's part indices -- equal its own run."""
    from paper_2410_04349_b200 import run_partitions

    monkeypatch.setenv("RB_MIXED", mixed)
    rel, path, _ = goldens.load("citation")
    n = len(rel)
    rng = np.random.default_rng(5)
    perm = rng.permutation(n)
    parts, at = [], 0
    for size in [900, 3, 1200, 2, 17, 5, 800, 40, 2, 9]:
        parts.append(DataPartition(len(parts), tuple(int(x) for x in perm[at:at + size])))
        at += size
    cfg = EngineConfig(symmetric_mode=symmetric)
    got = run_partitions(parts, rel, path, cfg)
    for p, cs in zip(parts, got):
        one = run_partition(p, rel, path, cfg)
        assert sorted(cs.pairs) == sorted(one.pairs)
        assert cs.stats.total_comparisons() == one.stats.total_comparisons()


def test_learned_shape_replays_without_retries(monkeypatch):
    """A new program of an already-run shape (the public API builds its
    objects afresh each call) starts from what the first one learned: its
    first run replays the survivor ranges with no overflow re-run."""
    from paper_2410_04349_b200.encode import RelationEncoding

    monkeypatch.setenv("RB_SURV_MIN", "64")
    monkeypatch.delenv("RB_LEARN", raising=False)
    rel, path, cases = goldens.load("citation")
    enc = RelationEncoding(rel).prepare(path.predicate_table)
    p1 = PathProgram(path, enc)
    from paper_2410_04349_b200._lib import RB_SYMMETRIC

    rows1, st1 = p1.run_raw(None, len(rel), RB_SYMMETRIC)
    p2 = PathProgram(path, enc)
    rows2, st2 = p2.run_raw(None, len(rel), RB_SYMMETRIC)
    assert sorted(zip(*rows1)) == sorted(zip(*rows2))
    assert st1.survivors > 64
    assert st2.retries == 0


def test_run_crosses_with_implied_root_equal_plain(monkeypatch):
    """Cross blocks keyed on an equality root (config 5's shape): the batch
    runs regated with the root implied (engine.implied_slots_of ->
    rb_run_batch_implied); rows equal the plain plan's and the per-block runs."""
    from paper_2410_04349_b200 import run_crosses, synth
    from paper_2410_04349_b200.engine import PathProgram, implied_slots_of

    w = synth.linkage(60_000, seed=5)
    blk = w.enc.columns[w.enc.get(("codes", "block"))].data
    bslot = [k for k, p in enumerate(w.path.predicate_table) if p.comparator == "eq" and p.lhs_attr == "block"]
    assert bslot
    prog = PathProgram(w.path, w.enc)
    big = sorted(w.blocks, key=lambda b: -len(b[0]))[:40]
    from paper_2410_04349_b200._lib import RB_SYMMETRIC
    refs = np.concatenate([r for r, _ in big]).astype(np.int32)
    offs = np.zeros(len(big) + 1, dtype=np.int64)
    np.cumsum([len(r) for r, _ in big], out=offs[1:])
    splits = np.array([sp for _, sp in big], dtype=np.int64)
    plain, st0 = prog.run_batch(refs, offs, splits, RB_SYMMETRIC)
    imp, st1 = prog.run_batch(refs, offs, splits, RB_SYMMETRIC, implied=1 << bslot[0])
    assert st0.comparisons == st1.comparisons
    assert sorted(zip(*plain)) == sorted(zip(*imp))
    assert all(len(np.unique(blk[r])) == 1 for r, _ in big)  # every block shares its key
    # the Python API derives the implied slot from DataPartition.branch_id / key_group
    from paper_2410_04349_b200 import DataPartition
    path = w.path
    b = list(path.root_slots).index(bslot[0]) if bslot[0] in path.root_slots else None
    if b is not None:
        pairs = [(DataPartition(2 * k, tuple(r[:sp].tolist()), branch_id=b, key_group=f"v:{k}"),
                  DataPartition(2 * k + 1, tuple(r[sp:].tolist()), branch_id=b, key_group=f"v:{k}"))
                 for k, (r, sp) in enumerate(big)]
        assert implied_slots_of(path, [p for pr in pairs for p in pr]) == 1 << bslot[0]
        got = run_crosses(pairs, None, path, program=prog)
        for (r, sp), cs in zip(big, got):
            want = prog.run_raw(r, len(r), RB_SYMMETRIC, split=sp)[0]
            assert sorted(cs.pairs) == sorted((int(a), int(c), path.rule_ids[int(d)]) for a, c, d in zip(*want))


@pytest.mark.parametrize("name", goldens.pipeline_names())
def test_run_partitions_split_by_branch_root(name, monkeypatch):
    """run_partitions over the partitions of several equality-rooted
    branches: forced to split (engine.SPLIT_PAIRS = 0), every branch's
    batch runs with its root implied; each partition's rows equal its own
    run_partition."""
    import paper_2410_04349_b200.engine as eng
    from paper_2410_04349_b200 import run_partitions
    from paper_2410_04349_b200.pipeline import BandingConfig, iter_partitions

    rel, path, _ = goldens.load(name)
    parts = [p for p in iter_partitions(rel, path, 16, BandingConfig()) if len(p.tuple_refs) > 1]
    monkeypatch.setattr(eng, "SPLIT_PAIRS", 0)
    got = run_partitions(parts, rel, path)
    for p, cs in zip(parts, got):
        assert sorted(cs.pairs) == sorted(run_partition(p, rel, path).pairs)
