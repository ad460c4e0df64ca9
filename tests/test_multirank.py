"""Sharding one partition over ranks: equal-pair row splits,
exercised with world_size-2 gloo process groups on the CPU.  Each rank
evaluates its outer-row shard (with the CPU oracle here; the GPU path runs
the same shard through rb_run_partition_rows), and the gathered union must
equal the whole partition."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import goldens
from paper_2410_04349_b200.engine import split_rows_by_pairs


@pytest.mark.parametrize("n,parts", [(1, 1), (2, 2), (5, 2), (100, 3), (4591, 8), (1_000_000, 8)])
def test_split_covers_and_balances(n, parts):
    cuts = split_rows_by_pairs(n, parts)
    assert cuts[0][0] == 0 and cuts[-1][1] == n
    assert all(a[1] == b[0] for a, b in zip(cuts, cuts[1:]))
    pairs = [sum(n - 1 - i for i in range(lo, hi)) if n < 10000 else
             (hi - lo) * n - (hi * (hi + 1) - lo * (lo + 1)) // 2 for lo, hi in cuts]
    total = n * (n - 1) // 2
    assert sum(pairs) == total
    if total >= parts * n:
        assert max(pairs) - min(pairs) <= 2 * n  # each cut lands within one row of its goal


def test_split_asymmetric():
    cuts = split_rows_by_pairs(10, 3, symmetric=False)
    assert cuts == [(0, 3), (3, 7), (7, 10)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, name, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle
    from paper_2410_04349_b200.encode import RelationEncoding, compile_program

    rel, path, cases = goldens.load(name)
    enc = RelationEncoding(rel).prepare(path.predicate_table)
    prog = compile_program(path, enc)
    lo, hi = split_rows_by_pairs(len(rel), world)[rank]
    rows, cmp, _ = oracle.run(enc, prog, None, len(rel), row_lo=lo, row_hi=hi, flags=1)
    gathered = [None] * world
    dist.all_gather_object(gathered, (rows.tolist(), cmp))
    if rank == 0:
        out.put(gathered)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["citation", "random_052"])
def test_two_rank_shards_union_equals_whole(name):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    gathered = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rel, path, cases = goldens.load(name)
    case = cases[0]
    union = sorted((int(t), int(s), path.rule_ids[int(k)]) for rows, _ in gathered for t, s, k in rows)
    assert union == goldens.expected_rows(case)
    assert sum(c for _, c in gathered) == case["comparisons"]
