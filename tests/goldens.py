"""Load the golden fixtures (tests/golden/*.json.gz, made by make_golden.py
from the reference) into this package's types, and replay them."""

from __future__ import annotations

import glob
import gzip
import json
import os

import numpy as np

from paper_2410_04349_b200.encode import RelationEncoding, compile_program
from paper_2410_04349_b200.plan import path_from_dict
from paper_2410_04349_b200.relation import relation_from_rows

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def names() -> list[str]:
    """Engine-level fixtures (one run per case)."""
    return sorted(n for n in _all() if not n.startswith(("pipeline_", "ingest")))


def pipeline_names() -> list[str]:
    """Reference pipeline_run fixtures (partitioning + pulls + collect)."""
    return sorted(n for n in _all() if n.startswith("pipeline_"))


def _all() -> list[str]:
    return [os.path.basename(p)[: -len(".json.gz")] for p in glob.glob(os.path.join(GOLDEN, "*.json.gz"))]


def load(name: str):
    with gzip.open(os.path.join(GOLDEN, name + ".json.gz"), "rt") as fh:
        doc = json.load(fh)
    r = doc["relation"]
    rel = relation_from_rows(r["names"], r["kinds"], r["rows"])
    path = path_from_dict(doc["path"])
    return rel, path, doc["cases"]


def expected_rows(case) -> list:
    return [tuple(x) for x in case["expected"]]


def oracle_rows(rel, path, case):
    """Replay one case through the CPU oracle (a restatement of the
    reference engine); returns (sorted [(t, s, rule_id)], comparisons)."""
    from oracle import oracle

    enc = RelationEncoding(rel).prepare(path.predicate_table)
    prog = compile_program(path, enc)
    flags = (1 if case["symmetric"] else 0) | (2 if case["enumerate"] else 0)
    if case["left"] is not None:
        refs = np.array(case["left"] + case["right"], dtype=np.int32)
        rows, cmp, _ = oracle.run(enc, prog, refs, len(refs), split=len(case["left"]), flags=flags)
    else:
        refs = None if case["refs"] is None else np.array(case["refs"], dtype=np.int32)
        n = len(rel) if refs is None else len(refs)
        rows, cmp, _ = oracle.run(enc, prog, refs, n, flags=flags)
    out = dedup_rows([(int(a), int(b), int(k)) for a, b, k in rows], case["symmetric"], case["enumerate"])
    return sorted((a, b, path.rule_ids[k]) for a, b, k in out), cmp


def dedup_rows(rows, symmetric, enumerate_all):
    """engine.py:600-616 on (t, s, rule_index) rows."""
    if enumerate_all:
        return list(dict.fromkeys(rows))
    if symmetric:
        best = {}
        for t, s, k in rows:
            if (t, s) not in best or k < best[(t, s)]:
                best[(t, s)] = k
        return [(t, s, k) for (t, s), k in best.items()]
    return rows
