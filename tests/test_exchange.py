"""The exchange step of the multi-GPU collect (distributed.exchange_rows):
each rank's collected rows are re-distributed by tuple-id range, then
collected once more; the ranks' shards in rank order must equal the collect
of every rank's rows (the reference's collect, pipeline.py:407-421).
Exercised with gloo process groups of 2 and 3 ranks on CPU tensors; the GPU
path runs the same function over NCCL with rb_collect_device as the collect."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _collect_np(t, s, r):
    """pipeline.py:407-421 restated: lexsort, first row per (t, s)."""
    order = np.lexsort((r, s, t))
    t, s, r = t[order], s[order], r[order]
    keep = np.ones(len(t), dtype=bool)
    keep[1:] = (t[1:] != t[:-1]) | (s[1:] != s[:-1])
    return t[keep], s[keep], r[keep]


def _rows_of(rank, n_tuples, k, seed):
    rng = np.random.default_rng(seed * 100 + rank)
    t = rng.integers(0, n_tuples, size=k).astype(np.int32)
    s = rng.integers(0, n_tuples, size=k).astype(np.int32)
    r = rng.integers(0, 5, size=k).astype(np.int32)
    if k:  # rows every rank emits too (cross-branch duplicates)
        t[:3], s[:3] = [0, n_tuples // 2, n_tuples - 1], [1, 2, 3]
    return _collect_np(t, s, r)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n_tuples, k, seed, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch

    from paper_2410_04349_b200.distributed import exchange_rows, t_bounds

    mine = _rows_of(rank, n_tuples, k if rank != 1 else k // 3, seed)
    got = exchange_rows(tuple(torch.from_numpy(x) for x in mine), n_tuples)
    t, s, r = _collect_np(*(x.numpy() for x in got))
    lo, hi = t_bounds(n_tuples, world)[rank:rank + 2]
    ok_range = bool(((t >= lo) & (t < hi)).all())
    gathered = [None] * world
    dist.all_gather_object(gathered, (t.tolist(), s.tolist(), r.tolist(), ok_range))
    if rank == 0:
        out.put(gathered)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n_tuples,k", [(2, 1000, 5000), (3, 10_000_000, 20000), (2, 7, 40), (3, 1000, 0)])
def test_exchange_then_collect_equals_global_collect(world, n_tuples, k):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    seed = 7
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_tuples, k, seed, q)) for r in range(world)]
    for p in procs:
        p.start()
    gathered = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(g[3] for g in gathered)
    every = [_rows_of(r, n_tuples, k if r != 1 else k // 3, seed) for r in range(world)]
    want = _collect_np(*(np.concatenate([e[c] for e in every]) for c in range(3)))
    got = tuple(np.concatenate([np.asarray(g[c], dtype=np.int32) for g in gathered]) for c in range(3))
    for a, b in zip(got, want):
        assert np.array_equal(a, b)


def test_t_bounds_cover():
    from paper_2410_04349_b200.distributed import t_bounds

    for n in (0, 1, 7, 10_000_000):
        for w in (1, 2, 3, 8):
            b = t_bounds(n, w)
            assert b[0] == 0 and b[-1] == n and all(x <= y for x, y in zip(b, b[1:]))
