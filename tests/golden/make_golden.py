"""Generate the golden fixtures from the REFERENCE implementation.

Run in the build container, where the reference is importable read-only:

    python tests/golden/make_golden.py            # writes tests/golden/*.json.gz

Every expected row list below is produced by the reference engine itself
(``ruleblock.engine.run_partition`` / ``run_cross``,
pkg/src/ruleblock/engine.py:619-681) on a FROZEN ExecutionPath stored next
to it, so the fixtures replay deterministically where the reference is
absent (the GPU box).  Sources of the cases:

* products: the bundled demo relation + rules (pkg/src/ruleblock/datasets.py:17-96)
  with the plan of pkg/tests/test_plan.py:65-66 (COSTS/SPS); configurations
  from pkg/tests/test_engine.py:284-386 and test_partitioning.py:179-186.
* random_*: ``random_instance(seed)`` (datasets.py:128-181) under the
  ``suite_oracle`` configuration rotation (bench.py:77-119).
* citation: ``citation_benchmark`` (datasets.py:332-398), 4,591 tuples.
* grouped / skewed: ``grouped_workload`` / ``skewed_partition_workload`` at
  reduced size (long edit strings, low thresholds).
* edges: the float-boundary vectors of SURVEY.md §8c, constant-equality
  direction cases (§8a a7), cross-attribute fallback slots, non-ASCII text.
"""

from __future__ import annotations

import gzip
import json
import os
import random
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.environ.get("RB_REFERENCE", "/root/reference/pkg")
sys.path.insert(0, os.path.join(REF, "src"))
sys.path.insert(0, os.path.join(REF, "tests"))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from ruleblock.bench import FAST_PLANNER  # noqa: E402
from ruleblock.datasets import (  # noqa: E402
    CITATION_HEADER,
    citation_benchmark,
    grouped_workload,
    random_instance,
    rows_to_relation,
    skewed_partition_workload,
    write_products,
)
from ruleblock.engine import EngineConfig, run_cross, run_partition  # noqa: E402
from ruleblock.planner.plan import build_tree, compile_path, generate_plan, order_predicates, score_tree  # noqa: E402
from ruleblock.relation import DataPartition, Kind, Relation, Schema, TupleRecord, load_relation  # noqa: E402
from ruleblock.rules import parse_ruleset, predicate_universe  # noqa: E402

from paper_2410_04349_b200.plan import path_to_dict  # noqa: E402


def plan_with(rules, costs, sps):
    uni = predicate_universe(rules)
    return compile_path(score_tree(build_tree(rules, order_predicates(uni, costs, sps)), sps))


def uniform_plan(rules):
    uni = predicate_universe(rules)
    return plan_with(rules, {p: 0.5 for p in uni}, {p: 0.5 for p in uni})


def cell(v):
    if type(v).__name__ == "Missing":
        return None
    return v


def relation_doc(rel):
    return {
        "names": list(rel.schema.names),
        "kinds": [k.value for _, k in rel.schema.attributes],
        "rows": [[cell(v) for v in rec.values] for rec in rel.tuples],
    }


def case(rel, path, *, refs=None, left=None, right=None, symmetric=True, enumerate_=False, name=""):
    cfg = EngineConfig(num_blocks=2, n_t=16, symmetric_mode=symmetric, enumerate_witnesses=enumerate_)
    if left is not None:
        cs = run_cross(DataPartition(-2, tuple(left)), DataPartition(-3, tuple(right)), rel, path, cfg)
    else:
        refs = list(range(len(rel))) if refs is None else list(refs)
        cs = run_partition(DataPartition(0, tuple(refs)), rel, path, cfg)
    return {
        "name": name,
        "refs": None if refs is None or refs == list(range(len(rel))) else list(refs),
        "left": None if left is None else list(left),
        "right": None if right is None else list(right),
        "symmetric": symmetric,
        "enumerate": enumerate_,
        "comparisons": cs.stats.total_comparisons(),
        "expected": sorted([int(t), int(s), r] for t, s, r in cs.pairs),
    }


def write(name, rel, path, cases, **extra):
    doc = {"relation": relation_doc(rel), "path": path_to_dict(path), "cases": cases, **extra}
    with gzip.open(os.path.join(HERE, name + ".json.gz"), "wt") as fh:
        json.dump(doc, fh, separators=(",", ":"))
    n = sum(len(c["expected"]) for c in cases)
    print(f"{name}: {len(rel)} tuples, {len(cases)} cases, {n} expected rows")


def rel_from(names, kinds, rows):
    schema = Schema(attributes=tuple((n, Kind(k)) for n, k in zip(names, kinds)))
    from ruleblock.relation import MISSING

    return Relation(
        schema=schema,
        tuples=tuple(
            TupleRecord(tid=i, eid=None, values=tuple(MISSING if v is None else v for v in row))
            for i, row in enumerate(rows)
        ),
    )


def products(tmp):
    from test_plan import COSTS, SPS

    data, rules_path = write_products(tmp)
    rel = load_relation(data)
    rules = parse_ruleset(open(rules_path).read())
    path = plan_with(rules, COSTS, SPS)
    cases = [
        case(rel, path, name="default"),
        case(rel, path, enumerate_=True, name="enumerate"),
        case(rel, path, symmetric=False, name="asymmetric"),
        case(rel, path, symmetric=False, enumerate_=True, name="asymmetric_enumerate"),
        case(rel, path, refs=(4, 3, 2, 1, 0), name="reversed"),
        case(rel, path, refs=(3, 1), name="subset"),
        case(rel, path, left=(0, 1), right=(2, 3, 4), name="cross"),
        case(rel, path, left=(2, 3, 4), right=(0, 1), name="cross_swapped"),
        case(rel, path, left=(0, 1), right=(2, 3, 4), symmetric=False, name="cross_asym"),
    ]
    write("products", rel, path, cases)
    # config 1: the 2-predicate eq + jaccard rule phi2 alone
    phi2 = parse_ruleset(json.dumps([r for r in json.load(open(rules_path)) if r["id"] == "phi2"]))
    write("products_phi2", rel, uniform_plan(phi2), [case(rel, uniform_plan(phi2), name="phi2")])


def randoms(tmp, seeds):
    for seed in seeds:
        rows, doc = random_instance(seed)
        rel = rows_to_relation(rows, ["cat", "num", "stext", "ltext"], tmp, name=f"r{seed}.csv")
        rules = parse_ruleset(json.dumps(doc))
        path = generate_plan(rel, rules, FAST_PLANNER).path
        sym = seed % 5 != 4
        cases = [case(rel, path, symmetric=sym, name="suite_oracle")]
        if seed % 3 == 0:
            cases.append(case(rel, path, symmetric=sym, enumerate_=True, name="enumerate"))
        if seed % 4 == 1:
            rng = random.Random(seed)
            refs = list(range(len(rel)))
            rng.shuffle(refs)
            cases.append(case(rel, path, refs=refs[: max(2, len(refs) * 2 // 3)], name="shuffled_subset"))
            half = len(refs) // 2
            cases.append(case(rel, path, left=refs[:half], right=refs[half:], name="cross"))
        write(f"random_{seed:03d}", rel, path, cases, seed=seed)


def citation(tmp):
    rows, doc, _truth = citation_benchmark()
    rel = rows_to_relation(rows, CITATION_HEADER, tmp, name="citation.csv")
    rules = parse_ruleset(json.dumps(doc))
    path = uniform_plan(rules)
    write("citation", rel, path, [case(rel, path, name="whole")])


def grouped(tmp):
    rows, doc = grouped_workload(n_groups=30, group_size=12, text_len=200, seed=3, edit_threshold=0.8)
    rel = rows_to_relation(rows, ["group", "text"], tmp, name="grouped.csv")
    rules = parse_ruleset(json.dumps(doc))
    path = uniform_plan(rules)
    write("grouped", rel, path, [case(rel, path, name="whole")])
    rows, doc = skewed_partition_workload(n=1200, n_t=64, heavy_intervals=2, heavy_group_size=8,
                                          heavy_text_len=300, seed=11)
    rel = rows_to_relation(rows, ["group", "text"], tmp, name="skewed.csv")
    rules = parse_ruleset(json.dumps(doc))
    path = uniform_plan(rules)
    write("skewed", rel, path, [case(rel, path, name="whole")])
    # edit-only, low threshold: every pair goes to the exact interpreter
    rng = random.Random(5)
    base = ["".join(rng.choices("abcde ", k=rng.randint(20, 60))) for _ in range(8)]
    rows = []
    for k in range(160):
        t = list(rng.choice(base))
        for _ in range(rng.randint(0, 12)):
            t[rng.randrange(len(t))] = rng.choice("abcdef ")
        rows.append(["".join(t)])
    rel = rel_from(["text"], ["short_text"], rows)
    rules = parse_ruleset(json.dumps([{"id": "e", "when": [
        {"t_attr": "text", "op": "sim", "s_attr": "text", "measure": "edit", "threshold": 0.55}]}]))
    path = uniform_plan(rules)
    write("edit_low", rel, path, [case(rel, path, name="whole"), case(rel, path, symmetric=False, name="asym")])


def edges():
    # (1) SURVEY §8c float edge: edit delta=0.3, "a"*27 vs "a"*90 -- the engine
    # rejects ((1-0.3)*90 = 62.99999999999999 < 63), the scorer would accept.
    rel = rel_from(["s"], ["short_text"], [["a" * 27], ["a" * 90], ["a" * 64], ["b" * 90], [None], [""], [""]])
    rules = parse_ruleset(json.dumps([{"id": "e", "when": [
        {"t_attr": "s", "op": "sim", "s_attr": "s", "measure": "edit", "threshold": 0.3}]}]))
    path = uniform_plan(rules)
    write("edge_edit_float", rel, path, [case(rel, path, name="sym"), case(rel, path, symmetric=False, name="asym")])

    # (2) SURVEY §8c float edge: jaccard delta=0.55, a 55-token subset of 100 tokens
    toks = [f"w{k}" for k in range(100)]
    rel = rel_from(["t"], ["long_text"], [[" ".join(toks)], [" ".join(toks[:55])], [" ".join(toks[:56])],
                                          [" ".join(toks[:54])], [" ".join(toks[45:])], [""], [None]])
    rules = parse_ruleset(json.dumps([{"id": "j", "when": [
        {"t_attr": "t", "op": "sim", "s_attr": "t", "measure": "jaccard", "threshold": 0.55}]}]))
    path = uniform_plan(rules)
    write("edge_jaccard_float", rel, path, [case(rel, path, name="sym")])

    # (3) direction: t.cat = 'c1' reads t only
    rel = rel_from(["cat", "x"], ["short_text", "short_text"], [["c1", "a"], ["c2", "a"], ["c1", "a"], [None, "a"]])
    rules = parse_ruleset(json.dumps([{"id": "k", "when": [
        {"t_attr": "cat", "op": "eq", "const": "c1"}, {"t_attr": "x", "op": "eq", "s_attr": "x"}]}]))
    path = uniform_plan(rules)
    write("edge_direction", rel, path, [
        case(rel, path, refs=(0, 1, 2), name="forward"),
        case(rel, path, refs=(2, 1, 0), name="reversed"),
        case(rel, path, refs=(1, 0, 3, 2), name="mixed"),
        case(rel, path, symmetric=False, name="asym"),
        case(rel, path, left=(1, 3), right=(0, 2), name="cross"),
    ])

    # (4) cross-attribute slots: text/text eq (shared dictionary), numeric/text
    # eq (mixed parse), cross jaccard / exact_token (shared vocabulary, no
    # prefilter), cross edit ASCII vs non-ASCII (different widths)
    rows = [
        ["12", 12.0, "Grand Hotel", "grand  hotel", "Zoë Smith", "zoe smith"],
        ["007", 7.0, "hotel grand", "Hotel, Grand!", "zoe smith", "Zoe Smith"],
        ["abc", 3.5, "grand", "grand", "ann", "anne"],
        ["3.5", None, "", "x", "", ""],
        [None, 12.0, "Grand Hotel Plaza", "plaza grand hotel", "bób", "bob"],
        ["$1,200", 1200.0, "a b c d", "d c b a", "anne", "ann"],
    ]
    rel = rel_from(["code", "num", "ta", "tb", "pa", "pb"],
                   ["short_text", "numeric", "short_text", "short_text", "short_text", "short_text"], rows)
    rules = parse_ruleset(json.dumps([
        {"id": "eqx", "when": [{"t_attr": "code", "op": "eq", "s_attr": "num"}]},
        {"id": "eqt", "when": [{"t_attr": "ta", "op": "eq", "s_attr": "tb"}]},
        {"id": "jx", "when": [{"t_attr": "ta", "op": "sim", "s_attr": "tb", "measure": "jaccard", "threshold": 0.6}]},
        {"id": "xx", "when": [{"t_attr": "ta", "op": "sim", "s_attr": "tb", "measure": "exact_token", "threshold": 1.0}]},
        {"id": "ex", "when": [{"t_attr": "pa", "op": "sim", "s_attr": "pb", "measure": "edit", "threshold": 0.7}]},
        {"id": "nc", "when": [{"t_attr": "num", "op": "eq", "const": 12}]},
    ]))
    path = uniform_plan(rules)
    write("edge_cross_attr", rel, path, [
        case(rel, path, name="sym"),
        case(rel, path, symmetric=False, name="asym"),
        case(rel, path, symmetric=False, enumerate_=True, name="asym_enum"),
    ])

    # (5) non-ASCII edit on one column (uint32 codepoints) and casefold
    rel = rel_from(["n"], ["short_text"], [["Straße"], ["STRASSE"], ["strasse"], ["Ελλάδα"], ["ελλαδα"],
                                          ["ΕΛΛΆΔΑ"], ["  MÜNCHEN "], ["münchen"], ["munchen"]])
    rules = parse_ruleset(json.dumps([{"id": "u", "when": [
        {"t_attr": "n", "op": "sim", "s_attr": "n", "measure": "edit", "threshold": 0.8}]}]))
    path = uniform_plan(rules)
    write("edge_unicode", rel, path, [case(rel, path, name="sym")])


def pipelines(tmp):
    """Reference pipeline_run (pipeline.py:245-433) on frozen plans:
    partitioning + every partition + optional sibling pulls + collect."""
    from ruleblock.partitioning import BandingConfig
    from ruleblock.pipeline import PipelineConfig, make_devices, pipeline_run
    from ruleblock.planner.plan import PlanBundle

    def bundle_for(rel, rules):
        b = generate_plan(rel, rules, FAST_PLANNER)
        return b

    jobs = []
    rows, doc, _ = citation_benchmark(n_tuples=1200, n_matches=500)
    jobs.append(("pipeline_citation", rows_to_relation(rows, CITATION_HEADER, tmp, name="pc.csv"), doc))
    for seed in (3, 7, 12):
        rows, doc = random_instance(seed)
        jobs.append((f"pipeline_random_{seed:03d}", rows_to_relation(rows, ["cat", "num", "stext", "ltext"], tmp,
                                                                     name=f"pr{seed}.csv"), doc))
    for name, rel, doc in jobs:
        rules = parse_ruleset(json.dumps(doc))
        bundle = bundle_for(rel, rules)
        cases = []
        for max_size, pulls, sym in ((32, False, True), (32, True, True), (8, True, True), (16, False, False)):
            res = pipeline_run(rel, rules, PipelineConfig(async_mode=False, max_partition_size=max_size,
                                                          enable_pulls=pulls, banding=BandingConfig(rows=4, seed=0)),
                               EngineConfig(num_blocks=1, symmetric_mode=sym), make_devices(2), plan=bundle)
            cases.append({"name": f"max{max_size}_pulls{int(pulls)}_sym{int(sym)}", "max_partition_size": max_size,
                          "enable_pulls": pulls, "symmetric": sym, "n_partitions": res.n_partitions,
                          "expected": sorted([int(t), int(s), r] for t, s, r in res.candidates.pairs)})
        doc_out = {"relation": relation_doc(rel), "path": path_to_dict(bundle.path), "cases": cases}
        with gzip.open(os.path.join(HERE, name + ".json.gz"), "wt") as fh:
            json.dump(doc_out, fh, separators=(",", ":"))
        print(f"{name}: {len(rel)} tuples, {[c['n_partitions'] for c in cases]} partitions, "
              f"{[len(c['expected']) for c in cases]} rows")


def main():
    # the suite_oracle rotation covers seeds 0..99 (bench.py:77-119)
    seeds = range(int(os.environ.get("RB_GOLDEN_SEED_LO", "0")), int(os.environ.get("RB_GOLDEN_SEEDS", "100")))
    if os.environ.get("RB_GOLDEN_ONLY") == "randoms":
        with tempfile.TemporaryDirectory() as tmp:
            randoms(tmp, seeds)
        return
    if os.environ.get("RB_GOLDEN_ONLY") == "pipelines":
        with tempfile.TemporaryDirectory() as tmp:
            pipelines(tmp)
        return
    with tempfile.TemporaryDirectory() as tmp:
        products(tmp)
        edges()
        randoms(tmp, seeds)
        grouped(tmp)
        if os.environ.get("RB_GOLDEN_SKIP_CITATION") != "1":
            citation(tmp)
        pipelines(tmp)


if __name__ == "__main__":
    main()
