"""Benchmark of the rule-evaluation hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step evaluates every unordered tuple pair of one synthetic 1M-tuple
citation-style relation (BASELINE config 2: 3 rules mixing equality, token
Jaccard and edit distance) as ONE partition -- 499,999,500,000
pairs -- and emits the surviving (t, s, rule) rows.

* value   -- pairs / s over the timed steps, inputs resident in HBM, timed
             with CUDA events on the stream the engine launches on, max over
             ranks.  L2 is flushed (a 512 MiB write) between timed steps.
* e2e     -- the same metric through the C ABI with HOST buffers: every step
             uploads the encoded relation and the program (H2D), evaluates,
             and copies the result rows back (D2H).
* roofline-- SURVEY §8d streaming-bytes model for the pair kernel.
* cpu_baseline -- the CPU oracle (a C restatement of the reference engine,
             oracle/rb_oracle.c) on a bounded row sample on this host's cores;
             the same rows are also checked for bit-exact parity against the GPU.

Multi-GPU (torchrun): weak scaling -- every rank evaluates its own 1M-tuple
partition (seed + rank), no data-path collective; NCCL only reduces the
timings and the row counts at the end.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "tuple pairs evaluated/sec and blocking wall-time at 1/2/4/8 B200 vs CPU ref"
WORKLOAD_DESC = {
    "citation3": "BASELINE config 2: 3 rules mixing eq, jaccard and edit",
    "edit_heavy": "BASELINE config 3: edit-distance-heavy rules, 64-256-char strings, maxd 2-5",
    "linkage": "BASELINE config 5: two-table linkage, Zipf(1.3) blocks, one cross run per block, batched",
    "citation3_parts": "config 2 relation in 512-tuple partitions (the reference pipeline's default), batched",
    "citation_small": "BASELINE config 1: the reference's citation_benchmark (4,591 tuples) with its frozen plan",
    "person5": "BASELINE config 4 (ii): person relation, 5 rules, data-aware plan, one partition",
    "person5_parts": "BASELINE config 4 (i): person relation, 5 rules, the pipeline's plan-derived partitions "
                     "(max_partition_size 65536) plus sibling pulls, batched",
}
UNIT = "pairs/s"


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            f = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except (ValueError, IndexError):
                continue
            for k, nm in enumerate(names):
                if len(f) > 3 + k and f[3 + k].lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def pinned_rows(k):
    """Three reusable pinned int32 host arrays of k rows (t, s, rule)."""
    import torch

    return tuple(torch.empty(max(1, k), dtype=torch.int32, pin_memory=True).numpy() for _ in range(3))


def pin_array(a):
    """A pinned (page-locked) host copy of a numpy array."""
    import torch

    t = torch.empty(a.nbytes, dtype=torch.uint8, pin_memory=True)
    out = t.numpy().view(a.dtype).reshape(a.shape)
    out[...] = a
    return out


def pinned_encoding(enc):
    """A copy of an Encoded whose column arrays live in pinned (page-locked)
    host memory, so the H2D copies of the e2e leg run at DMA speed."""
    from paper_2410_04349_b200.encode import Column, Encoded

    def pin(a):
        return None if a is None else pin_array(a)

    pe = Encoded(enc.n)
    pe.columns = [Column(c.kind, pin(c.data), pin(c.offsets), pin(c.missing)) for c in enc.columns]
    pe.index = dict(enc.index)
    return pe


def algorithmic_bytes_per_pair(enc, path, evals_frac, rows_per_pair):
    """A = sum_s E_s * b_s + C * 10 B, per pair.  E_s/pairs comes
    from the oracle's exact first-touch counts on the sample rows."""
    from paper_2410_04349_b200.encode import SLOT_EDIT, SLOT_EQ_CODE, SLOT_EXACT, SLOT_JACCARD

    total = 0.0
    terms = {}
    for s, p in enumerate(path.predicate_table):
        kind, _, rc, _ = enc.slot_for(p)
        col = enc.columns[rc]
        if kind == SLOT_EQ_CODE:
            b = 4.0
        elif kind in (SLOT_JACCARD, SLOT_EXACT):
            b = 4.0 + 4.0 * float(np.diff(col.offsets).mean())
        elif kind == SLOT_EDIT:
            b = 4.0 + float(np.diff(col.offsets).mean()) * col.width
        else:
            b = 0.0
        terms[p.describe()] = {"evals_per_pair": float(evals_frac[s]), "bytes": b}
        total += float(evals_frac[s]) * b
    return total + 10.0 * rows_per_pair, terms


def cpu_sample(w, prog, rows, nthreads):
    """Oracle on outer rows `rows` (list of (lo, hi)); returns rows, pairs, seconds, evals."""
    from oracle import oracle

    out, pairs, evals, secs = [], 0, np.zeros(prog.n_slots, dtype=np.int64), 0.0
    for lo, hi in rows:
        t0 = time.perf_counter()
        r, cmp, ev = oracle.run(w.enc, prog, None, w.n, row_lo=lo, row_hi=hi, flags=1, nthreads=nthreads)
        secs += time.perf_counter() - t0
        out.append(r)
        pairs += cmp
        evals += ev
    return np.concatenate(out) if out else np.zeros((0, 3), np.int64), pairs, secs, evals


def sample_rows(n, budget_pairs, k=8):
    """k disjoint row slices spread over the triangle whose pairs sum to
    ~budget; the whole triangle when it is within budget."""
    if n * (n - 1) // 2 <= budget_pairs:
        return [(0, n)]
    per = max(1, budget_pairs // k)
    out = []
    for q in range(k):
        lo = int(q * n / k)
        nxt = int((q + 1) * n / k)
        rows = max(1, per // max(1, n - lo - 1))
        out.append((lo, min(nxt, lo + rows)))
    return out


def ncu_capture(w, pairs_step):
    """(dram bytes per launch, pipe utilisation) of the committed ncu capture
    of this workload at this size (profiles/traffic.json), or (None, None)."""
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "traffic.json")
    pipe = None
    if os.path.exists(tfile):
        try:  # ncu dram__bytes_read.sum + dram__bytes_write.sum per launch, same workload and size
            entry = json.load(open(tfile)).get(w.name, {})
            if entry.get("n") == w.n:
                traffic = entry.get("bytes_per_launch")
                m = entry.get("metrics", {})
                pipe = {k: float(m[k]["value"]) for k in (
                    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
                    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
                    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
                    "smsp__issue_active.avg.pct_of_peak_sustained_active") if k in m}
                if "smsp__inst_executed.sum" in m:  # the per-pair instruction cost of the capture
                    pipe["warp_instructions_per_pair"] = float(m["smsp__inst_executed.sum"]["value"]) / pairs_step
                pipe["source"] = entry.get("capture")
                # the busiest issue pipe of the capture: the kernel's speed-of-light fraction
                # (the inner tuples are reused from shared memory, so DRAM is not the bound)
                names = {"sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "ALU",
                         "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "XU",
                         "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "shared memory"}
                busiest = max((k for k in names if k in pipe), key=lambda k: pipe[k], default=None)
                if busiest:
                    pipe["binding"] = {"pipe": names[busiest], "frac": pipe[busiest] / 100.0}
        except Exception:
            traffic = None
    return traffic, pipe


def blocks_cpu_parity(w, prog, budget, kms, pairs_step, n_rows):
    """Block workloads: oracle on a seeded sample of whole blocks (CPU
    baseline), the same blocks re-run on the GPU for bit-exact parity."""
    from oracle import oracle
    from paper_2410_04349_b200._lib import RB_SYMMETRIC

    rng = np.random.default_rng(0)
    order = rng.permutation(len(w.blocks))
    chosen, pairs = [], 0
    for k in order:
        refs, sp = w.blocks[k]
        c = sp * (len(refs) - sp) if sp >= 0 else len(refs) * (len(refs) - 1) // 2
        if c > budget // 4 or pairs + c > budget:
            continue
        chosen.append(k)
        pairs += c
    cores = os.cpu_count() or 1
    secs, cmp_total, ok = 0.0, 0, True
    evals = np.zeros(prog.n_slots, dtype=np.int64)
    sub = [w.blocks[k] for k in chosen]
    refs = np.concatenate([r for r, _ in sub]).astype(np.int32)
    offs = np.zeros(len(sub) + 1, dtype=np.int64)
    np.cumsum([len(r) for r, _ in sub], out=offs[1:])
    (gt, gs, gr, gp), _ = prog.run_batch(refs, offs, np.array([sp for _, sp in sub], dtype=np.int64), RB_SYMMETRIC)
    got = sorted(zip(gp.tolist(), gt.tolist(), gs.tolist(), gr.tolist()))
    want = []
    for bi, (r, sp) in enumerate(sub):
        t0 = time.perf_counter()
        rows, cmp, ev = oracle.run(w.enc, prog.program, r, len(r), split=sp, flags=1, nthreads=cores)
        secs += time.perf_counter() - t0
        cmp_total += cmp
        evals += ev
        want += [(bi, int(a), int(b), int(c)) for a, b, c in rows]
    ok = sorted(want) == got
    cpu = {"value": cmp_total / secs, "unit": UNIT, "cores": cores, "kind": "port",
           "sample": f"{len(sub)} whole cross blocks, {cmp_total} pairs (oracle/rb_oracle.c, OpenMP {cores} threads)"}
    parity = {"blocks_checked": len(sub), "rows_checked": len(want), "pairs_checked": cmp_total, "bit_exact": ok}
    peak, peak_kind = measured_peak()
    bpp, terms = algorithmic_bytes_per_pair(w.enc, w.path, evals / max(1, cmp_total), n_rows / max(1, pairs_step))
    k_ms = float(np.mean(kms))
    achieved = bpp * pairs_step / (k_ms / 1e3) / 1e9
    traffic, pipe = ncu_capture(w, pairs_step)
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": traffic, "ncu_pipes": pipe, "peak_kind": peak_kind, "bytes_per_pair": bpp, "kernel_ms": k_ms, "terms": terms,
            "model": "SURVEY 8d streaming bytes: sum_s E_s*b_s + 10 B per row; E_s from oracle first-touch counts"}
    return cpu, parity, roof


def run_reference_blocks(args, w, prog, cores, world):
    from oracle import oracle

    rng = np.random.default_rng(0)
    chosen, pairs = [], 0
    for k in rng.permutation(len(w.blocks)):
        refs, sp = w.blocks[k]
        c = sp * (len(refs) - sp) if sp >= 0 else len(refs) * (len(refs) - 1) // 2
        if c <= args.cpu_pairs // 4 and pairs + c <= args.cpu_pairs:
            chosen.append(k)
            pairs += c
    secs = cmp = 0
    for it in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        c_it = 0
        for k in chosen[: (4 if it < args.warmup else None)]:
            refs, sp = w.blocks[k]
            _, c, _ = oracle.run(w.enc, prog, refs, len(refs), split=sp, flags=1, nthreads=cores)
            c_it += c
        if it >= args.warmup:
            secs += time.perf_counter() - t0
            cmp += c_it
    v = cmp / secs
    total = w.pairs()
    line = {
        "metric": METRIC, "value": v, "unit": UNIT, "impl": "reference", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": {"workload": f"{w.name} n={w.n} ({WORKLOAD_DESC.get(w.name, w.name)}), {len(w.blocks)} blocks",
                   "pairs_per_step_full": total, "sample_pairs_per_step": cmp // args.steps},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{len(chosen)} whole cross blocks, {cmp // args.steps} pairs per step"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "blocking_wall_s_full_extrapolated": total / v,
    }
    print(json.dumps(line), flush=True)


def run_reference(args, rank, world):
    """--impl reference: the reference CPU engine restated in C (oracle), all
    host threads, bounded sample per step; rank 0 only."""
    if rank != 0:
        return
    from paper_2410_04349_b200 import synth
    from paper_2410_04349_b200.encode import compile_program

    w = synth.WORKLOADS[args.workload](args.n, seed=args.seed)
    prog = compile_program(w.path, w.enc)
    cores = os.cpu_count() or 1
    if w.blocks is not None:
        return run_reference_blocks(args, w, prog, cores, world)
    rows = sample_rows(w.n, args.cpu_pairs)
    for _ in range(args.warmup):
        cpu_sample(w, prog, rows[:1], cores)
    pairs = secs = 0
    for _ in range(args.steps):
        _, p, s, _ = cpu_sample(w, prog, rows, cores)
        pairs += p
        secs += s
    v = pairs / secs
    total_pairs = w.n * (w.n - 1) // 2
    line = {
        "metric": METRIC, "value": v, "unit": UNIT, "impl": "reference", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": {"workload": f"{w.name} n={w.n} ({WORKLOAD_DESC.get(w.name, w.name)}), one symmetric partition",
                   "pairs_per_step_full": total_pairs, "sample_pairs_per_step": pairs // args.steps},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{len(rows)} outer-row slices, {pairs // args.steps} pairs per step; "
                                   f"full step extrapolates to {total_pairs / v:.0f} s"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "blocking_wall_s_full_extrapolated": total_pairs / v,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="citation3")
    ap.add_argument("--tuples", dest="n", type=int, default=1_000_000, help="tuples per GPU")
    ap.add_argument("--seed", type=int, default=2024)
    ap.add_argument("--cpu-pairs", type=int, default=120_000_000, help="oracle sample size (pairs)")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    rank, world, local = dist_env()
    if args.warmup < 3:
        args.warmup = 3

    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    ndev = max(1, torch.cuda.device_count())
    dev = local % ndev
    torch.cuda.set_device(dev)
    # one rank per GPU over NCCL; ranks sharing a GPU (functional tests on a
    # 1-GPU box) reduce over gloo instead
    backend = "nccl" if world <= ndev else "gloo"
    red_dev = "cuda" if backend == "nccl" else "cpu"
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group("gloo")

    from paper_2410_04349_b200 import synth
    from paper_2410_04349_b200._lib import RB_SYMMETRIC
    from paper_2410_04349_b200.engine import DeviceRelation, PathProgram, context

    w = synth.WORKLOADS[args.workload](args.n, seed=args.seed + rank)
    ctx = context(dev)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    prog = PathProgram(w.path, w.enc, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    if w.blocks is not None:  # many cross blocks / partitions: one batched launch per step
        b_refs = pin_array(np.concatenate([r for r, _ in w.blocks]).astype(np.int32))  # the batch's input refs
        b_offs = np.zeros(len(w.blocks) + 1, dtype=np.int64)
        np.cumsum([len(r) for r, _ in w.blocks], out=b_offs[1:])
        b_splits = np.array([sp for _, sp in w.blocks], dtype=np.int64)

        def step(p, host=True):
            (t, s, r, _), st_ = p.run_batch(b_refs, b_offs, b_splits, RB_SYMMETRIC,
                                            out=None if host_rows is None else host_rows + (host_part,))
            return (t, s, r), st_
    elif world > 1 and backend == "nccl":
        # N GPUs: each rank evaluates its partition, then the final collect is
        # one NCCL all-gather of the row counts and of the rows themselves,
        # straight from the device result buffers (distributed.gather_rows)
        from paper_2410_04349_b200.distributed import gather_rows, run_rows_device

        gathered = [0]

        def step(p, host=False):
            rows_d, st_ = run_rows_device(p, None, w.n, RB_SYMMETRIC, 0, w.n)
            allrows = gather_rows(rows_d)
            gathered[0] = int(allrows.shape[0])
            if host:  # the e2e leg reads the collected rows back
                allrows.cpu()
            return (rows_d[:, 0], rows_d[:, 1], rows_d[:, 2]), st_
    else:
        def step(p, host=True):
            return p.run_raw(None, w.n, RB_SYMMETRIC, out=host_rows)

    # result rows land in reusable pinned host buffers (sized by the first run)
    host_rows = None
    rows, st = step(prog)
    host_rows = pinned_rows(len(rows[0]))
    host_part = pinned_rows(len(rows[0]))[0]
    for _ in range(args.warmup - 1):
        rows, st = step(prog)
    n_rows = len(rows[0])
    pairs_step = int(st.comparisons)

    times, kms, vms = [], [], []
    sampler = ClockSampler(dev)
    with sampler:
        for _ in range(args.steps):
            flush.fill_(1)
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            h0 = time.perf_counter()
            e0.record(stream)
            rows, st = step(prog)
            e1.record(stream)
            torch.cuda.synchronize()
            h1 = time.perf_counter()
            times.append(e0.elapsed_time(e1))
            kms.append(st.pair_ms if st.pair_ms > 0 else st.kernel_ms)  # the dominant (pair) kernel
            vms.append(st.kernel_ms - kms[-1])  # deferred verification kernel
            print(f"step: events {times[-1]:.1f} ms, kernels {st.kernel_ms:.1f} ms (pair {kms[-1]:.1f}), "
                  f"host {1e3 * (h1 - h0):.1f} ms, "
                  f"survivors {st.survivors}, rows {len(rows[0])}, launches {st.launches}, retries {st.retries}",
                  file=sys.stderr)
            assert st.comparisons == pairs_step and len(rows[0]) == n_rows
    barrier()
    t_total = torch.tensor([sum(times)], dtype=torch.float64, device=red_dev)
    counts = torch.tensor([pairs_step * args.steps, n_rows], dtype=torch.float64, device=red_dev)
    if world > 1:
        dist.all_reduce(t_total, op=dist.ReduceOp.MAX)
        dist.all_reduce(counts, op=dist.ReduceOp.SUM)
    ms_step = t_total.item() / args.steps
    value = counts[0].item() / (t_total.item() / 1e3)

    # ---- e2e: host buffers through the C ABI, copies inside the timed region.
    # The step's inputs (the encoded columns) sit in pinned host memory, as a
    # loader would leave them; pinning happens once, outside the timed region.
    e2e_steps = args.e2e_steps or max(1, min(args.steps, 3))
    host_enc = pinned_encoding(w.enc)
    h2d = sum(c.data.nbytes + (0 if c.offsets is None else c.offsets.nbytes)
              + (0 if c.missing is None else c.missing.nbytes) for c in w.enc.columns)
    h2d += prog.program.tables.nbytes + prog.program.slots.nbytes + 4 * 4 * len(prog.program.ins_op)
    # one untimed pass first: the stream-ordered pool grows to the e2e working set once
    drel = DeviceRelation(ctx, host_enc)
    p2 = PathProgram(w.path, host_enc, compiled=prog.program, drel=drel)
    step(p2)
    p2.close()
    drel.close()
    barrier()
    t0 = time.perf_counter()
    phase = {"upload": 0.0, "program": 0.0, "run": 0.0, "free": 0.0}
    for _ in range(e2e_steps):
        q0 = time.perf_counter()
        drel = DeviceRelation(ctx, host_enc)  # H2D of every encoded column
        q1 = time.perf_counter()
        p2 = PathProgram(w.path, host_enc, compiled=prog.program, drel=drel)  # H2D of the program
        q2 = time.perf_counter()
        rows2, st2 = step(p2, host=True)  # evaluate + D2H of the rows
        q3 = time.perf_counter()
        print(f"e2e step: kernels {st2.kernel_ms:.1f} ms (pair {st2.pair_ms:.1f}), launches {st2.launches}, "
              f"retries {st2.retries}", file=sys.stderr)
        assert len(rows2[0]) == n_rows
        p2.close()
        drel.close()
        q4 = time.perf_counter()
        for k, v in zip(phase, (q1 - q0, q2 - q1, q3 - q2, q4 - q3)):
            phase[k] += v / e2e_steps
    print("e2e phases (s): " + ", ".join(f"{k} {v:.4f}" for k, v in phase.items()), file=sys.stderr)
    torch.cuda.synchronize()
    e2e_s = torch.tensor([(time.perf_counter() - t0) / e2e_steps], dtype=torch.float64, device=red_dev)
    if world > 1:
        dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
    e2e_value = counts[0].item() / args.steps / e2e_s.item()
    nccl_collect = world > 1 and backend == "nccl" and w.blocks is None
    d2h = 12 * (gathered[0] if nccl_collect else n_rows) + 8 * 68

    # ---- CPU oracle sample (rank 0, N = 1): baseline + parity on the same rows
    cpu = None
    parity = None
    roof = None
    peak, peak_kind = measured_peak()
    if rank == 0 and world == 1 and not args.no_cpu and w.blocks is not None:
        cpu, parity, roof = blocks_cpu_parity(w, prog, args.cpu_pairs, kms, pairs_step, n_rows)
    elif rank == 0 and world == 1 and not args.no_cpu:
        cores = os.cpu_count() or 1
        srows = sample_rows(w.n, args.cpu_pairs)
        orc_rows, orc_pairs, orc_s, orc_evals = cpu_sample(w, prog.program, srows, cores)
        cpu = {"value": orc_pairs / orc_s, "unit": UNIT, "cores": cores, "kind": "port",
               "sample": f"{len(srows)} outer-row slices of the same relation, {orc_pairs} pairs "
                         f"(oracle/rb_oracle.c, OpenMP {cores} threads)"}
        ok = True
        for lo, hi in srows:
            (gt, gs, gr), gst = prog.run_raw(None, w.n, RB_SYMMETRIC, row_lo=lo, row_hi=hi)
            sel = (orc_rows[:, 0] >= lo) & (orc_rows[:, 0] < hi)
            want = sorted(map(tuple, orc_rows[sel].tolist()))
            got = sorted(zip(gt.tolist(), gs.tolist(), gr.tolist()))
            ok &= want == got
        parity = {"rows_checked": int(len(orc_rows)), "pairs_checked": int(orc_pairs), "bit_exact": bool(ok)}
        # every row of the last timed step: a true match (refs = identity, so t is the
        # lower tid), carrying the oracle's first witness, no pair twice
        from oracle import oracle as _orc

        at, as_, ar = (np.asarray(x) for x in rows)
        wit = _orc.witness(w.enc, prog.program, at, as_, nthreads=cores)
        key = at.astype(np.int64) * w.n + as_
        parity["all_step_rows"] = {"rows": int(len(at)), "witness_exact": bool((wit == ar).all()),
                                   "ordered": bool((at < as_).all()), "distinct": bool(len(np.unique(key)) == len(key)),
                                   "check": "oracle.witness on every emitted (t, s): rule == oracle first witness"}
        bpp, terms = algorithmic_bytes_per_pair(w.enc, w.path, orc_evals / max(1, orc_pairs), n_rows / pairs_step)
        k_ms = float(np.mean(kms))
        achieved = bpp * pairs_step / (k_ms / 1e3) / 1e9
        traffic, pipe = ncu_capture(w, pairs_step)
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "peak_kind": peak_kind,
                "true_bound": "integer pipes: XU (POPC) and ALU issue (inner tuples are reused from shared "
                              "memory, so DRAM is not the limit; see DESIGN.md 3.1)",
                "ncu_pipes": pipe,
                "model": "SURVEY 8d streaming bytes: sum_s E_s*b_s + 10 B per row; E_s from oracle first-touch counts",
                "bytes_per_pair": bpp, "kernel_ms": k_ms, "verify_kernel_ms": float(np.mean(vms)),
                "kernel": "rb_pair_kernel_spec (phase 1; CUDA events on the engine's stream)", "terms": terms}

    clocks = sampler.summary()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int32", "data": "synthetic",
            "config": {"workload": f"{w.name} n={w.n} per GPU ({WORKLOAD_DESC.get(w.name, w.name)}), "
                                   + (f"{len(w.blocks)} blocks in one batched launch per GPU" if w.blocks is not None
                                      else "one symmetric partition per GPU"),
                       "pairs_per_step_per_gpu": pairs_step, "rows_per_step_per_gpu": n_rows,
                       "l2": "flushed (512 MiB write) between timed steps", "parallelism": f"partition-per-gpu x{world}",
                       "collective": (f"{backend}: all-gather of row counts and rows (final collect)"
                                      if world > 1 and backend == "nccl" and w.blocks is None
                                      else backend if world > 1 else None)},
            "blocking_wall_s": ms_step / 1e3,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                    "blocking_wall_s": e2e_s.item()},
            "roofline": roof, "cpu_baseline": cpu, "parity": parity,
            "gpu_launches": int(st.launches) * args.steps,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
