"""The device half of pipeline_run (csrc/rb_pipeline.cu): partitioning,
the LPT split of the units over ranks, and collect -- each against its host
restatement of the reference (pipeline.iter_partitions /
sibling_pull_pairs / collect, themselves pinned to the reference in
test_partitioning.py and test_pipeline.py)."""

import numpy as np
import pytest

import goldens
from paper_2410_04349_b200 import EngineConfig
from paper_2410_04349_b200.engine import CandidateSet, PathProgram
from paper_2410_04349_b200.encode import RelationEncoding
from paper_2410_04349_b200.pipeline import (
    BandingConfig,
    branch_order,
    collect,
    iter_partitions,
    partition_keys,
    partition_on_device,
    rank_keys,
    sibling_pull_pairs,
)

NAMES = goldens.pipeline_names()


def test_rank_keys_follow_sorted_key_strings():
    keys = ["v:b", "\x00missing", "n:10.0", "v:b", "n:2.0", "b:1a:3", "b:2:0"]
    ranks, distinct = rank_keys(keys)
    assert distinct == sorted(set(keys))
    assert [distinct[r] for r in ranks] == keys
    assert ranks[1] == 0  # the missing key sorts first


def test_branch_order_puts_equality_first():
    rel, path, _ = goldens.load(NAMES[0])
    order = branch_order(path)
    roots = [path.predicate_table[s] for s in path.root_slots]
    assert sorted(order) == list(range(len(roots)))
    eq = [b for b in order if roots[b].comparator == "eq"]
    assert order[: len(eq)] == eq


def _program(rel, path):
    enc = RelationEncoding(rel).prepare(path.predicate_table)
    return PathProgram(path, enc)


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("maxp", [1, 3, 16, 512])
@pytest.mark.parametrize("pulls", [False, True])
def test_device_partitions_equal_iter_partitions(name, maxp, pulls):
    rel, path, _ = goldens.load(name)
    prog = _program(rel, path)
    kb = partition_keys(rel, path, BandingConfig())
    parts = partition_on_device(prog, keys=np.stack([k for _, k, _ in kb]), branch_ids=[b for b, _, _ in kb],
                                max_partition_size=maxp, pulls=pulls, key_groups={b: g for b, _, g in kb})
    want = list(iter_partitions(rel, path, maxp, BandingConfig()))
    got = parts.partitions()
    assert [(p.pid, p.tuple_refs, p.branch_id, p.key_group, p.sibling_group) for p in got] == \
           [(p.pid, p.tuple_refs, p.branch_id, p.key_group, p.sibling_group) for p in want]
    assert parts.n_pulls == (len(sibling_pull_pairs(want)) if pulls else 0)
    if pulls:
        assert parts.pulls() == sibling_pull_pairs(want)


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("world", [1, 2, 3, 7])
@pytest.mark.parametrize("symmetric", [True, False])
def test_rank_shares_partition_the_units(name, world, symmetric):
    """The union of every rank's rows equals the per-partition runs (host
    collect), and the ranks' comparison counts add up."""
    rel, path, _ = goldens.load(name)
    prog = _program(rel, path)
    kb = partition_keys(rel, path, BandingConfig())
    parts = partition_on_device(prog, keys=np.stack([k for _, k, _ in kb]), branch_ids=[b for b, _, _ in kb],
                                max_partition_size=8, pulls=True)
    cfg = EngineConfig(symmetric_mode=symmetric)
    rows, cmp = [], 0
    for rank in range(world):
        res = prog.run_parts(parts, cfg.flags(), rank, world)
        t, s, r = res.copy()
        cmp += int(res.stats().comparisons)
        rows.append(CandidateSet(arrays=(t.astype(np.int64), s.astype(np.int64), r.astype(np.int64)),
                                 rule_ids=path.rule_ids))
        res.close()
    from paper_2410_04349_b200 import run_cross, run_partitions

    ps = parts.partitions()
    want_sets = run_partitions(ps, rel, path, cfg, program=prog)
    by = {p.pid: p for p in ps}
    want_sets += [run_cross(by[a], by[b], rel, path, cfg, program=prog) for a, b in parts.pulls()]
    want_cmp = sum(c.stats.total_comparisons() for c in want_sets)
    assert cmp == want_cmp
    assert sorted(collect(rows, path.rule_ids).pairs) == sorted(collect(want_sets, path.rule_ids).pairs)


def _collect_np(t, s, r):
    order = np.lexsort((r, s, t))
    t, s, r = t[order], s[order], r[order]
    keep = np.ones(len(t), dtype=bool)
    keep[1:] = (t[1:] != t[:-1]) | (s[1:] != s[:-1])
    return t[keep], s[keep], r[keep]


@pytest.mark.gpu
@pytest.mark.parametrize("n_tuples,n_rules,k", [(10, 1, 0), (10, 1, 1), (1000, 3, 5000), (10_000_000, 5, 300_000),
                                                (2_000_000_000, 64, 200_000), (2**31 - 1, 3, 1000)])
def test_device_collect_equals_lexsort(n_tuples, n_rules, k):
    import torch

    from paper_2410_04349_b200 import _lib
    from paper_2410_04349_b200.engine import context

    rng = np.random.default_rng(k + n_rules)
    hi = min(n_tuples, 3000)  # dense enough for duplicate (t, s) across rules
    t = rng.integers(0, hi, size=k).astype(np.int32)
    s = rng.integers(0, hi, size=k).astype(np.int32)
    if n_tuples > hi and k:
        t[::7] = n_tuples - 1 - rng.integers(0, 5, size=len(t[::7]))
    r = rng.integers(0, n_rules, size=k).astype(np.int32)
    dev = torch.device("cuda", 0)
    cols = [torch.from_numpy(x).to(dev) for x in (t, s, r)]
    out = [torch.empty(max(1, k), dtype=torch.int32, device=dev) for _ in range(3)]
    torch.cuda.synchronize()
    cnt = _lib.ctypes.c_int64(-1)
    _lib.check(_lib.lib().rb_collect_device(context(0).handle, *[_lib.c_vp(x.data_ptr()) for x in cols], k, n_tuples,
                                            n_rules, *[_lib.c_vp(x.data_ptr()) for x in out], _lib.ctypes.byref(cnt)))
    got = tuple(x[: cnt.value].cpu().numpy() for x in out)
    want = _collect_np(t.astype(np.int64), s.astype(np.int64), r.astype(np.int64))
    assert cnt.value == len(want[0])
    for a, b in zip(got, want):
        assert np.array_equal(a, b)


@pytest.mark.gpu
@pytest.mark.parametrize("n", [30_000, 200_000])
def test_implied_root_regating_keeps_the_candidate_set(n, monkeypatch):
    """rb_run_parts evaluates the branch holding most pairs with its
    equality root implied (rb::choose_gate): the same collected rows and
    comparison counts as the plain filter plan (RB_IMPLIED_OFF)."""
    from paper_2410_04349_b200 import synth
    from paper_2410_04349_b200.pipeline import PipelineConfig, run_pipeline_encoded, root_predicates

    w = synth.person5(n, seed=4)
    roots = root_predicates(w.path)
    bids = branch_order(w.path)
    cols = [w.enc.get(("codes", roots[b].lhs_attr)) for b in bids]
    cfg = PipelineConfig(max_partition_size=4096 if n > 50_000 else 512, enable_pulls=True,
                         single_partition_threshold=0)
    out = []
    for off, eq_any in (("1", "0"), (None, "0"), (None, "1")):
        monkeypatch.setenv("RB_EQ_ANY", eq_any)  # the OR-first equality stage of the regated plan (opt-in)
        if off:
            monkeypatch.setenv("RB_IMPLIED_OFF", off)
        else:
            monkeypatch.delenv("RB_IMPLIED_OFF", raising=False)
        res = run_pipeline_encoded(w.enc, w.path, cfg, EngineConfig(), code_cols=cols, branch_ids=bids)
        out.append((res.candidates.arrays, res.candidates.stats.total_comparisons()))
        res.parts.close()
    (a, ca) = out[0]
    for b, cb in out[1:]:
        assert ca == cb
        for x, y in zip(a, b):
            assert np.array_equal(x, y)
    assert len(a[0]) > 0
