"""BASELINE config 2 at full size against ONE COMPLETE oracle run.

tests/golden/citation3_full.json holds the row count, per-rule counts and
the sha256 of the sorted (t, s, rule) rows of oracle/rb_oracle.c over every
one of the 499,999,500,000 pairs of synth.citation3(1M, seed 2024) as one
symmetric partition (tools/full_oracle_citation3.py, CPU-hours, once).  The
GPU's complete output must hash to the same digest: recall and precision
over the whole pair space, not a sample."""

import hashlib
import json
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "citation3_full.json")


def _doc():
    if not os.path.exists(GOLDEN):
        pytest.skip("tests/golden/citation3_full.json not generated (tools/full_oracle_citation3.py)")
    return json.load(open(GOLDEN))


def test_golden_is_consistent():
    doc = _doc()
    assert doc["pairs"] == 1_000_000 * 999_999 // 2
    assert sum(doc["rows_per_rule"].values()) == doc["rows"]
    assert len(doc["sha256_sorted_t_s_rule_int32le"]) == 64


@pytest.mark.gpu
def test_gpu_complete_output_matches_full_oracle_digest():
    doc = _doc()
    from paper_2410_04349_b200 import synth
    from paper_2410_04349_b200._lib import RB_SYMMETRIC
    from paper_2410_04349_b200.engine import PathProgram

    w = synth.citation3(1_000_000, seed=2024)
    assert list(w.path.rule_ids) == doc["path_rule_ids"]
    prog = PathProgram(w.path, w.enc)
    (t, s, r), st = prog.run_raw(None, w.n, RB_SYMMETRIC)
    assert int(st.comparisons) == doc["pairs"]
    rows = np.stack([t, s, r], axis=1).astype("<i4")
    rows = rows[np.lexsort((rows[:, 2], rows[:, 1], rows[:, 0]))]
    assert len(rows) == doc["rows"]
    assert {w.path.rule_ids[k]: int((rows[:, 2] == k).sum()) for k in range(len(w.path.rule_ids))} == \
        doc["rows_per_rule"]
    assert hashlib.sha256(np.ascontiguousarray(rows).tobytes()).hexdigest() == doc["sha256_sorted_t_s_rule_int32le"]
