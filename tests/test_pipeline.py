"""pipeline_run (partitioning + every partition + sibling pulls + collect)
against the reference's own pipeline_run output on frozen plans
(tests/golden/pipeline_*.json.gz, made by make_golden.py)."""

import numpy as np
import pytest

import goldens
from paper_2410_04349_b200 import EngineConfig
from paper_2410_04349_b200.pipeline import (
    BandingConfig,
    PipelineConfig,
    collect,
    iter_partitions,
    pipeline_run,
    sibling_pull_pairs,
)

NAMES = goldens.pipeline_names()


def test_pipeline_fixtures_present():
    assert len(NAMES) >= 4


@pytest.mark.parametrize("name", NAMES)
def test_pipeline_logic_with_the_oracle(name):
    """CPU: our partitions + pulls + collect, each partition evaluated by
    the oracle, reproduce the reference pipeline exactly."""
    from oracle import oracle
    from paper_2410_04349_b200.encode import RelationEncoding, compile_program
    from paper_2410_04349_b200.engine import CandidateSet

    rel, path, cases = goldens.load(name)
    enc = RelationEncoding(rel).prepare(path.predicate_table)
    prog = compile_program(path, enc)
    for case in cases:
        sym = case["symmetric"]
        parts = list(iter_partitions(rel, path, case["max_partition_size"], BandingConfig()))
        if len(rel) <= case["max_partition_size"]:
            pytest.skip("single-partition case")
        assert len(parts) == case["n_partitions"]
        sets = []
        blocks = [(np.array(p.tuple_refs, np.int32), -1) for p in parts if len(p.tuple_refs) > 1 or not sym]
        if case["enable_pulls"]:
            by = {p.pid: p for p in parts}
            blocks += [(np.array(by[a].tuple_refs + by[b].tuple_refs, np.int32), len(by[a].tuple_refs))
                       for a, b in sibling_pull_pairs(parts)]
        for refs, split in blocks:
            rows, _, _ = oracle.run(enc, prog, refs, len(refs), split=split, flags=1 if sym else 0)
            sets.append(CandidateSet(arrays=(rows[:, 0], rows[:, 1], rows[:, 2]), rule_ids=path.rule_ids))
        got = sorted(collect(sets, path.rule_ids).pairs)
        assert got == goldens.expected_rows(case), case["name"]


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("devices", [(0,), (0, 0)])
def test_pipeline_run_matches_reference(name, devices):
    rel, path, cases = goldens.load(name)
    for case in cases:
        res = pipeline_run(rel, path,
                           PipelineConfig(max_partition_size=case["max_partition_size"],
                                          enable_pulls=case["enable_pulls"], devices=devices),
                           EngineConfig(symmetric_mode=case["symmetric"]))
        assert res.n_partitions == case["n_partitions"]
        assert sorted(res.candidates.pairs) == goldens.expected_rows(case), case["name"]
