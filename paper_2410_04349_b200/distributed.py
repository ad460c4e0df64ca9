"""One partition sharded over the ranks of a process group, one GPU per rank
(the reference's process-per-device pipeline, pipeline.py:177-209,
re-done over real GPUs).

The pair space of a partition is cut into contiguous outer-row ranges of
equal pair count (``split_rows_by_pairs``); rank r evaluates its range with
``rb_run_partition_rows`` -- no data exchange while evaluating.  The only
collective is the final gather the north star names: an all-gather of the
per-rank row counts, then of the (t, s, rule) rows themselves, straight from
the device result buffers (``rb_result_device``) over NCCL, so every rank
ends with the whole candidate set without a host round trip.

Each pair is evaluated on exactly one rank, so the union is already what
``_dedup_witnesses`` (engine.py:600-616) returns for one partition.
"""

from __future__ import annotations

import time
from typing import Optional

import numpy as np

from . import _lib
from ._lib import check, lib
from .engine import (BlockStats, CandidateSet, EngineConfig, PathProgram, RunStats, _program_for, _refs_array,
                     split_rows_by_pairs)
from .errors import ConfigError


class _DevRows:
    """__cuda_array_interface__ view of one int32 device array."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<i4", "data": (ptr, False), "version": 3,
                                         "strides": None}


def run_rows_device(prog: PathProgram, refs, n: int, flags: int, row_lo: int, row_hi: int):
    """Evaluate outer rows [row_lo, row_hi) and return the rows as one
    (k, 3) int32 torch tensor on the program's device (t, s, rule), plus the
    run's rb_stats."""
    import torch

    L = lib()
    res = _lib.c_vp()
    refs_a = None if refs is None else _lib.i32(refs)
    check(L.rb_run_partition_rows(prog.ctx.handle, prog.drel.handle, prog.handle, _lib.ptr(refs_a), n, row_lo,
                                  row_hi, flags, _lib.ctypes.byref(res)))
    try:
        cnt = _lib.ctypes.c_int64(0)
        check(L.rb_result_count(res, _lib.ctypes.byref(cnt)))
        k = cnt.value
        dev = torch.device("cuda", prog.ctx.device)
        out = torch.empty((k, 3), dtype=torch.int32, device=dev)
        if k:
            pt, ps, pr = _lib.c_vp(), _lib.c_vp(), _lib.c_vp()
            check(L.rb_result_device(res, _lib.ctypes.byref(pt), _lib.ctypes.byref(ps), _lib.ctypes.byref(pr), None))
            for col, p in enumerate((pt, ps, pr)):  # the run has completed (its count is on the host)
                out[:, col].copy_(torch.as_tensor(_DevRows(p.value, k), device=dev))
            # the copies ran on torch's stream: finish them before the library
            # frees or reuses the result buffers on its own stream
            torch.cuda.current_stream(dev).synchronize()
        st = _lib.RbStats()
        check(L.rb_result_stats(res, _lib.ctypes.byref(st)))
    finally:
        L.rb_result_destroy(res)
    return out, st


def gather_rows(rows, group=None):
    """All-gather variable-length (k_r, 3) int32 row blocks: first the
    counts, then the rows padded to the largest count, one collective each.
    Returns the concatenation in rank order (every rank gets the same)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    if rows.is_cuda and dist.get_backend(group) == "gloo":  # ranks sharing one GPU (functional runs)
        return gather_rows(rows.cpu(), group).to(rows.device)
    cnt = torch.tensor([rows.shape[0]], dtype=torch.int64, device=rows.device)
    counts = torch.empty(world, dtype=torch.int64, device=rows.device)
    dist.all_gather_into_tensor(counts, cnt, group=group)
    counts_h = counts.tolist()
    kmax = max(counts_h)
    if kmax == 0:
        return rows[:0]
    padded = torch.zeros((kmax, 3), dtype=rows.dtype, device=rows.device)
    padded[: rows.shape[0]] = rows
    everything = torch.empty((world * kmax, 3), dtype=rows.dtype, device=rows.device)
    dist.all_gather_into_tensor(everything, padded, group=group)
    return torch.cat([everything[r * kmax: r * kmax + c] for r, c in enumerate(counts_h)])


def run_partition_distributed(partition, relation, path, cfg: Optional[EngineConfig] = None, reg=None,
                              encoded=None, program=None, group=None) -> CandidateSet:
    """``run_partition`` over every rank of ``group`` (default: the world),
    one GPU per rank (``LOCAL_RANK``).  Collective: every rank must call it
    with the same arguments; every rank returns the whole CandidateSet."""
    import torch.distributed as dist

    cfg = EngineConfig.of(cfg)
    if partition is None or len(partition.tuple_refs) == 0:
        return CandidateSet(pairs=[])
    if not dist.is_initialized():
        raise ConfigError("run_partition_distributed needs an initialised torch.distributed process group")
    started = time.perf_counter()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    prog = _program_for(path, relation, reg, encoded, program)
    refs = _refs_array(partition)
    n = len(refs)
    lo, hi = split_rows_by_pairs(n, world, symmetric=cfg.symmetric_mode)[rank]
    rows, st = run_rows_device(prog, refs, n, cfg.flags(), lo, hi)
    allrows = gather_rows(rows, group).cpu().numpy().astype(np.int64)
    import torch

    stats_t = torch.tensor([int(st.comparisons), int(st.survivors), int(st.emitted)], dtype=torch.int64,
                           device=rows.device)
    dist.all_reduce(stats_t, group=group)
    cmp, surv, emitted = stats_t.tolist()
    block = BlockStats(block_id=0, intervals_processed=max(1, -(-n // cfg.n_t)), comparisons=cmp,
                       busy_s=st.kernel_ms / 1e3, slot_evals=np.zeros(prog.n_slots, dtype=np.int64),
                       emitted=emitted, survivors=surv)
    stats = RunStats(blocks=[block], wall_s=time.perf_counter() - started, n_intervals=max(1, -(-n // cfg.n_t)),
                     kernel_ms=float(st.kernel_ms), launches=int(st.launches), specialized=bool(st.specialized),
                     jit_log=prog.jit_log)
    return CandidateSet(stats=stats, arrays=(allrows[:, 0], allrows[:, 1], allrows[:, 2]), rule_ids=prog.rule_ids)


def t_bounds(n_tuples: int, world: int) -> list:
    """Rank r owns the rows whose t lies in [bounds[r], bounds[r+1])."""
    return [(n_tuples * r) // world for r in range(world + 1)]


def exchange_rows(rows, n_tuples: int, group=None):
    """The exchange step of the multi-GPU collect: (t, s, rule) int32 rows,
    sorted by t (a rank's collected rows), are re-distributed so that rank r
    receives every rank's rows with t in its tuple-id range (``t_bounds``).
    One all-to-all of the per-destination counts, one of the rows packed
    (k, 3).  Returns this rank's received (t, s, rule), the senders' runs
    back to back in rank order.  Works on CUDA tensors over NCCL and on CPU
    tensors over gloo."""
    import torch
    import torch.distributed as dist

    t, s, r = rows
    world = dist.get_world_size(group)
    if world == 1:
        return t, s, r
    if t.is_cuda and dist.get_backend(group) == "gloo":  # ranks sharing one GPU (functional runs)
        got = exchange_rows((t.cpu(), s.cpu(), r.cpu()), n_tuples, group)
        return tuple(x.to(t.device) for x in got)
    dev = t.device
    inner = torch.tensor(t_bounds(n_tuples, world)[1:-1], dtype=t.dtype, device=dev)
    cuts = torch.searchsorted(t, inner)  # t is sorted: each destination is a contiguous run
    edges = torch.cat([torch.zeros(1, dtype=torch.int64, device=dev), cuts.to(torch.int64),
                       torch.tensor([t.shape[0]], dtype=torch.int64, device=dev)])
    send = edges[1:] - edges[:-1]
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send, group=group)
    send_h, recv_h = send.tolist(), recv.tolist()
    packed = torch.stack([t, s, r], dim=1)
    out = torch.empty((sum(recv_h), 3), dtype=t.dtype, device=dev)
    dist.all_to_all_single(out, packed, output_split_sizes=recv_h, input_split_sizes=send_h, group=group)
    return out[:, 0].contiguous(), out[:, 1].contiguous(), out[:, 2].contiguous()
