"""The multi-rank path of distributed.py on the CPU: world_size-2 gloo
process groups.  gather_rows (count all-gather + padded row all-gather) and
the equal-pair row shards must reassemble exactly the single-device result;
each rank's shard is evaluated by the oracle here (the GPU path runs the
same shard through rb_run_partition_rows, tests/test_gpu_parity.py)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import goldens
from paper_2410_04349_b200.distributed import gather_rows
from paper_2410_04349_b200.engine import split_rows_by_pairs


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _run(world, target, args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, q) + args) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(out, key=lambda x: x[0])


def _gather_worker(rank, world, port, q, sizes):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    k = sizes[rank]
    rows = torch.arange(3 * k, dtype=torch.int32).reshape(k, 3) + 1000 * rank
    got = gather_rows(rows)
    q.put((rank, got.numpy().tolist()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("sizes", [(3, 5), (0, 4), (0, 0), (7, 0)])
def test_gather_rows_two_ranks(sizes):
    out = _run(2, _gather_worker, (sizes,))
    want = []
    for r, k in enumerate(sizes):
        want += (np.arange(3 * k).reshape(k, 3) + 1000 * r).tolist()
    for _, got in out:
        assert got == want


def _shard_worker(rank, world, port, q, name, symmetric):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle
    from paper_2410_04349_b200.encode import RelationEncoding, compile_program

    rel, path, cases = goldens.load(name)
    enc = RelationEncoding(rel).prepare(path.predicate_table)
    prog = compile_program(path, enc)
    lo, hi = split_rows_by_pairs(len(rel), world, symmetric=symmetric)[rank]
    rows, cmp, _ = oracle.run(enc, prog, None, len(rel), row_lo=lo, row_hi=hi, flags=1 if symmetric else 0)
    allrows = gather_rows(torch.as_tensor(np.asarray(rows, dtype=np.int32).reshape(-1, 3)))
    q.put((rank, allrows.numpy().tolist(), cmp))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["citation", "random_052"])
@pytest.mark.parametrize("symmetric", [True, False])
def test_shards_gathered_equal_whole(name, symmetric):
    out = _run(2, _shard_worker, (name, symmetric))
    rel, path, cases = goldens.load(name)
    case = {"symmetric": symmetric, "enumerate": False, "refs": None, "left": None, "right": None}
    want, cmp = goldens.oracle_rows(rel, path, case)
    for _, rows, _ in out:
        got = sorted((t, s, path.rule_ids[k]) for t, s, k in rows)
        assert got == want
    assert sum(c for _, _, c in out) == cmp


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["citation", "products"])
def test_distributed_single_rank_nccl(name):
    """The device path of run_partition_distributed on one GPU: rows from
    rb_result_device, NCCL all-gathers (world size 1 on a 1-GPU box)."""
    from paper_2410_04349_b200 import DataPartition, EngineConfig
    from paper_2410_04349_b200.distributed import run_partition_distributed

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        rel, path, cases = goldens.load(name)
        for case in cases:
            if case["left"] is not None or case["enumerate"]:
                continue
            refs = tuple(range(len(rel))) if case["refs"] is None else tuple(case["refs"])
            cfg = EngineConfig(symmetric_mode=case["symmetric"])
            cs = run_partition_distributed(DataPartition(0, refs), rel, path, cfg)
            assert sorted(cs.pairs) == goldens.expected_rows(case)
            assert cs.stats.total_comparisons() == case["comparisons"]
    finally:
        dist.destroy_process_group()
