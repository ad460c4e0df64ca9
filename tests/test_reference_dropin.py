"""The drop-in claim on the reference's OWN objects, run live beside it.

The reference package (``ruleblock``) is installed test-only under
baseline/_ref (``pip install --target baseline/_ref``, git-ignored; it
travels to the GPU box with the snapshot) or read from /root/reference in the
build container.  The package under test never imports it.

* CPU: the encoder accepts the reference's Relation / ExecutionPath / config
  objects as produced by its own loaders and planner.
* GPU: the reference's own scenarios -- pkg/tests/test_engine.py:283-392 (the
  products relation, reversed refs, asymmetric mode, enumerate witnesses,
  coverage counts), pkg/tests/test_partitioning.py:161-186 (cross pulls), the
  suite_oracle rotation over 100 random_instance seeds (bench.py:77-119) --
  with the reference's run_partition / run_cross swapped for this package's
  (module attributes monkeypatched, so the reference's own callers such as
  pipeline.cross_partition_pull reach the GPU engine), compared with the
  reference engine itself and its nested-loop oracle on the same objects.
"""

import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for cand in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
    if os.path.isdir(os.path.join(cand, "ruleblock")):
        sys.path.append(cand)
        break
rb = pytest.importorskip("ruleblock", reason="the reference package is not installed (baseline/_ref)")

import ruleblock.bench as rbench  # noqa: E402
import ruleblock.engine as rengine  # noqa: E402
import ruleblock.pipeline as rpipeline  # noqa: E402
from ruleblock.datasets import random_instance, rows_to_relation, write_products  # noqa: E402
from ruleblock.planner.plan import generate_plan  # noqa: E402
from ruleblock.relation import DataPartition, load_relation  # noqa: E402
from ruleblock.rules import parse_ruleset  # noqa: E402

import paper_2410_04349_b200 as ours  # noqa: E402

FAST = rbench.FAST_PLANNER
# the reference's own entry points, kept before any test swaps them
REF_RUN_PARTITION = rengine.run_partition
REF_PIPELINE_RUN = rpipeline.pipeline_run


@pytest.fixture(scope="module")
def products(tmp_path_factory):
    data, rules_path = write_products(tmp_path_factory.mktemp("products"))
    relation = load_relation(data)
    rules = parse_ruleset(rules_path.read_text())
    path = generate_plan(relation, rules, FAST).path
    return relation, rules, path


@pytest.fixture
def swapped(monkeypatch):
    """The reference's engine entry points replaced by this package's."""
    for mod in (rengine, rpipeline):
        monkeypatch.setattr(mod, "run_partition", ours.run_partition)
        monkeypatch.setattr(mod, "run_cross", ours.run_cross)
    return ours


def _rows(cs):
    return sorted(cs.pairs)


def test_reference_objects_encode(products):
    from paper_2410_04349_b200.encode import RelationEncoding, compile_program

    relation, _, path = products
    enc = RelationEncoding(relation).prepare(list(path.predicate_table))
    prog = compile_program(path, enc, rb.measures.default_registry())
    assert prog.n_slots == len(path.predicate_table)
    assert ours.EngineConfig.of(rengine.EngineConfig(symmetric_mode=False, n_t=7)).flags() & 1 == 0


@pytest.mark.gpu
def test_products_scenarios_equal_reference(products, swapped):
    relation, rules, path = products
    whole = DataPartition(pid=0, tuple_refs=tuple(range(5)))
    cases = [
        (whole, rengine.EngineConfig(num_blocks=2, n_t=2, n_w=2)),
        (whole, rengine.EngineConfig(num_blocks=1, n_t=5)),
        (whole, rengine.EngineConfig(num_blocks=2, n_t=2, symmetric_mode=False)),
        (DataPartition(pid=0, tuple_refs=(4, 3, 2, 1, 0)), rengine.EngineConfig(num_blocks=1, n_t=2)),
        (whole, rengine.EngineConfig(num_blocks=1, enumerate_witnesses=True)),
    ]
    for part, cfg in cases:
        got = swapped.run_partition(part, relation, path, cfg)
        want = REF_RUN_PARTITION(part, relation, path, cfg)
        assert _rows(got) == _rows(want), cfg
        assert got.stats.total_comparisons() == want.stats.total_comparisons()
    cs = swapped.run_partition(whole, relation, path, rengine.EngineConfig(num_blocks=2, n_t=2, n_w=2))
    assert cs.pair_set() == {(0, 3), (0, 4), (3, 4), (1, 2)}  # test_engine.py:284-291
    rev = swapped.run_partition(DataPartition(pid=0, tuple_refs=(4, 3, 2, 1, 0)), relation, path)
    assert all(t < s for t, s, _ in rev.pairs) and rev.pair_set() == cs.pair_set()  # :359-364
    assert len(swapped.run_partition(None, relation, path)) == 0  # :388-390


@pytest.mark.gpu
def test_cross_pull_through_reference_caller(products, swapped):
    """pkg/tests/test_partitioning.py:179-186, via the reference's own
    cross_partition_pull (pipeline.py:242) reaching the GPU run_cross."""
    relation, _, path = products
    left = DataPartition(pid=0, tuple_refs=(0, 1), branch_id=0)
    right = DataPartition(pid=1, tuple_refs=(2, 3, 4), branch_id=0)
    cs = rpipeline.cross_partition_pull(left, right, relation, path, rengine.EngineConfig(num_blocks=2, n_t=1))
    assert isinstance(cs, ours.CandidateSet)  # the GPU engine answered
    assert cs.stats.total_comparisons() == 2 * 3
    assert cs.pair_set() == {(0, 3), (0, 4), (1, 2)}


@pytest.mark.gpu
def test_suite_oracle_100_seeds_live(tmp_path):
    """bench.py:77-119's rotation over seeds 0..99: the GPU engine on the
    reference's relation and plan == the reference engine == its oracle."""
    ref_engine = rengine
    modes = ("off", "inter", "inter+intra")
    bad = []
    for seed in range(100):
        rows, doc = random_instance(seed)
        relation = rows_to_relation(rows, ["cat", "num", "stext", "ltext"], tmp_path, name=f"r{seed}.csv")
        rules = parse_ruleset(json.dumps(doc))
        sym = seed % 5 != 4
        cfg = ref_engine.EngineConfig(n_t=(16, 32, 64)[seed % 3], n_w=8, num_blocks=1 + seed % 3,
                                      lanes_per_block=(4, 32)[seed % 2], stealing=modes[seed % 3],
                                      symmetric_mode=sym, buffer_half_capacity=(1, 64, 4096)[seed % 3],
                                      chunk_size=(7, 64, 4096)[seed % 3])
        path = generate_plan(relation, rules, FAST).path
        part = DataPartition(pid=0, tuple_refs=tuple(range(len(relation))))
        got = ours.run_partition(part, relation, path, cfg)
        want = REF_RUN_PARTITION(part, relation, path, cfg)
        oracle = rbench.brute_force_candidates(relation, rules, symmetric=sym)
        if _rows(got) != _rows(want) or got.pair_set() != oracle:
            bad.append(seed)
        assert got.stats.total_comparisons() == want.stats.total_comparisons()
    assert bad == []


@pytest.mark.gpu
def test_pipeline_run_on_reference_objects_equals_reference(tmp_path):
    """This package's pipeline_run (partition + execute + collect on the
    GPU) on the reference's relation, rules and frozen PlanBundle == the
    reference's pipeline_run (pipeline.py:245-433) on the same objects."""
    ref_pipeline = rpipeline
    for seed in (3, 7, 12, 40):
        rows, doc = random_instance(seed)
        relation = rows_to_relation(rows, ["cat", "num", "stext", "ltext"], tmp_path, name=f"p{seed}.csv")
        rules = parse_ruleset(json.dumps(doc))
        bundle = generate_plan(relation, rules, FAST)
        for maxp, pulls in ((8, True), (16, False)):
            rcfg = ref_pipeline.PipelineConfig(async_mode=False, max_partition_size=maxp, enable_pulls=pulls)
            want = REF_PIPELINE_RUN(relation, rules, rcfg, rengine.EngineConfig(num_blocks=1),
                                             ref_pipeline.make_devices(1), plan=bundle)
            got = ours.pipeline_run(relation, rules, ours.PipelineConfig(max_partition_size=maxp, enable_pulls=pulls),
                                    plan=bundle)
            assert sorted(got.candidates.pairs) == sorted(want.candidates.pairs), (seed, maxp, pulls)
            assert got.n_partitions == want.n_partitions
