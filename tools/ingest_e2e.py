"""End-to-end blocking time from a CSV file (SURVEY §8d "end-to-end time"):
CSV -> load_relation (columnar ingest) -> encoding -> device upload ->
run_partition over one partition of every tuple -> CandidateSet.

    python tools/ingest_e2e.py [N] [--reference]

Writes an N-row citation-style CSV (title / authors / venue / year / cat)
to /tmp, plans the config-2 rules on a sample, and prints the time of each
stage.  --reference also times the reference's own load_relation on the
same file (needs /root/reference; only in the build container)."""

import csv
import json
import os
import random
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2410_04349_b200 import DataPartition, EngineConfig, ingest, run_partition  # noqa: E402
from paper_2410_04349_b200.encode import RelationEncoding  # noqa: E402
from paper_2410_04349_b200.engine import PathProgram  # noqa: E402
from paper_2410_04349_b200.rules import parse_ruleset, predicate_universe  # noqa: E402
from paper_2410_04349_b200.synth import CITATION3_RULES, data_aware_plan  # noqa: E402


def write_csv(path, n, seed=1):
    rng = random.Random(seed)
    words = [f"w{k}" for k in range(800)]
    names = [f"n{k}" for k in range(400)]
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["eid", "title", "authors", "venue", "year", "cat"])
        for i in range(n):
            w.writerow([f"e{i}", " ".join(rng.choices(words, k=rng.randint(6, 10))),
                        ", ".join(rng.choices(names, k=rng.randint(1, 3))), f"v{rng.randrange(10)}",
                        str(1995 + rng.randrange(16)), f"c{rng.randrange(1000)}"])


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 1_000_000
    path = f"/tmp/rb_ingest_{n}.csv"
    if not os.path.exists(path):
        write_csv(path, n)
    rules = parse_ruleset(json.dumps(CITATION3_RULES))
    t = {}
    t0 = time.perf_counter()
    rel = ingest.load_relation(path)
    t["ingest_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    enc = RelationEncoding(rel).prepare(sorted(predicate_universe(rules), key=str))
    t["encode_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    path_ = data_aware_plan(enc, rules, sample=200_000, seed=0)  # planning (not part of blocking time)
    t["plan_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    prog = PathProgram(path_, enc)
    t["upload_and_compile_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    cs = run_partition(DataPartition(0, tuple(range(n))), rel, path_, EngineConfig(), program=prog)
    t["run_s"] = time.perf_counter() - t0
    pairs = cs.stats.total_comparisons()
    total = t["ingest_s"] + t["encode_s"] + t["upload_and_compile_s"] + t["run_s"]
    out = {"n": n, "pairs": pairs, "rows": len(cs), **{k: round(v, 4) for k, v in t.items()},
           "blocking_s_from_csv": round(total, 4), "pairs_per_s_from_csv": pairs / total}
    if "--reference" in sys.argv:
        sys.path.insert(0, "/root/reference/pkg/src")
        from ruleblock.relation import load_relation as ref_load

        t0 = time.perf_counter()
        ref_load(path)
        out["reference_load_relation_s"] = round(time.perf_counter() - t0, 3)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
