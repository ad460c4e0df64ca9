"""The reference's own published benchmark suites, run through this
package's GPU engine on the reference's own objects, beside the reference
engine itself (its published times: pkg/test_output.txt:274 and :300).

* suite_stealing (pkg/src/ruleblock/bench.py:155-215): skewed_partition_
  workload(n=50_000) -- one whole partition, heavy groups of 900-character
  texts under an edit threshold of 0.55 (maxd[900] = 405): Myers'
  bit-vector path on the device.  Published: 23.8 s best of 3 (stealing on).
* suite_scaling (bench.py:267-313): grouped_workload(2000 x 50, 200-char
  texts, edit 0.8, perturb_divisor 3) through pipeline_run (2000 group
  partitions).  Published: 142.6 s on 1 device, 110.4 s on 8.

The relation, rules and frozen plan are built by the reference (installed
test-only under baseline/_ref; /root/reference in the build container).
Our run_partition / pipeline_run take those objects unchanged.  With
--reference the reference engine runs too, for pair-set parity and its
time on this host.  Writes one JSON line per suite.

    python tools/reference_suites.py [--reference] [--out FILE]
"""

import argparse
import json
import os
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
for cand in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
    if os.path.isdir(os.path.join(cand, "ruleblock")):
        sys.path.append(cand)
        break

import ruleblock.bench as rbench  # noqa: E402
import ruleblock.engine as rengine  # noqa: E402
import ruleblock.pipeline as rpipeline  # noqa: E402
from ruleblock.datasets import grouped_workload, skewed_partition_workload  # noqa: E402
from ruleblock.planner.plan import generate_plan  # noqa: E402

import paper_2410_04349_b200 as ours  # noqa: E402

PUBLISHED = {"suite_stealing": {"wall_s": 23.8283, "source": "pkg/test_output.txt:274 (stealing on, best of 3, 2 cores)"},
             "suite_scaling": {"wall_s_1_device": 142.5703, "wall_s_8_devices": 110.4429,
                               "source": "pkg/test_output.txt:300 (2 cores)"}}


def timed(fn, repeats):
    best, out = None, None
    for _ in range(repeats):
        t0 = time.perf_counter()
        out = fn()
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return out, best


def stealing(args, tmp):
    blocks = max(2, min(os.cpu_count() or 2, 8))
    rows, doc = skewed_partition_workload(n=50_000, n_t=256, n_w=1024, num_blocks=blocks, heavy_intervals=18,
                                          seed=11)
    relation, rules = rbench._load_instance(rows, doc, tmp, header=["group", "text"])
    bundle = generate_plan(relation, rules, rbench.FAST_PLANNER)
    part = rbench._whole_partition(relation)
    prog = ours.PathProgram(bundle.path, ours.RelationEncoding(relation).prepare(list(bundle.path.predicate_table)))
    ours.run_partition(part, relation, bundle.path, program=prog)  # JIT + pool warm-up
    cs, wall = timed(lambda: ours.run_partition(part, relation, bundle.path, program=prog), 3)
    line = {"suite": "suite_stealing", "n_tuples": len(relation), "pairs_evaluated": cs.stats.total_comparisons(),
            "candidates": len(cs), "gpu_wall_s": wall, "gpu_kernel_ms": cs.stats.kernel_ms,
            "gpu_pairs_per_s": cs.stats.total_comparisons() / wall, "published": PUBLISHED["suite_stealing"]}
    if args.reference:
        cfg = rengine.EngineConfig(n_t=256, n_w=1024, num_blocks=blocks, stealing="inter+intra", chunk_size=65536)
        want, rwall = timed(lambda: rengine.run_partition(part, relation, bundle.path, cfg), 1)
        line.update(reference_wall_s=rwall, reference_cores=os.cpu_count(), reference_blocks=blocks,
                    identical=sorted(cs.pairs) == sorted(want.pairs), speedup=rwall / wall)
    return line


def scaling(args, tmp):
    rows, doc = grouped_workload(n_groups=2000, group_size=50, seed=3, edit_threshold=0.8, perturb_divisor=3)
    relation, rules = rbench._load_instance(rows, doc, tmp, header=["group", "text"])
    bundle = generate_plan(relation, rules, rbench.FAST_PLANNER)
    cfg = ours.PipelineConfig(async_mode=True)
    ours.pipeline_run(relation, rules, cfg, plan=bundle)  # JIT + pool warm-up
    res, wall = timed(lambda: ours.pipeline_run(relation, rules, cfg, plan=bundle), 3)
    line = {"suite": "suite_scaling", "n_tuples": len(relation), "partitions": res.n_partitions,
            "pairs_evaluated": res.candidates.stats.total_comparisons(), "candidates": len(res.candidates),
            "gpu_wall_s": wall, "gpu_timings_s": res.timings, "published": PUBLISHED["suite_scaling"]}
    if args.reference:
        want, rwall = timed(lambda: rpipeline.pipeline_run(relation, rules, rpipeline.PipelineConfig(async_mode=True),
                                                           rengine.EngineConfig(num_blocks=1),
                                                           rpipeline.make_devices(1), plan=bundle), 1)
        line.update(reference_wall_s_1_device=rwall, reference_cores=os.cpu_count(),
                    identical=sorted(res.candidates.pairs) == sorted(want.candidates.pairs), speedup=rwall / wall)
    return line


def async_suite(args, tmp):
    """suite_async (bench.py:314-372): grouped_workload(600 x 40, 150-char
    texts), pipeline_run async vs sync on 4 simulated devices in the
    reference; ours: pipeline_run on the GPU (one device)."""
    rows, doc = grouped_workload(n_groups=600, group_size=40, text_len=150, seed=5, edit_threshold=0.8,
                                 perturb_divisor=3)
    relation, rules = rbench._load_instance(rows, doc, tmp, header=["group", "text"])
    bundle = generate_plan(relation, rules, rbench.FAST_PLANNER)
    cfg = ours.PipelineConfig(async_mode=True)
    ours.pipeline_run(relation, rules, cfg, plan=bundle)
    res, wall = timed(lambda: ours.pipeline_run(relation, rules, cfg, plan=bundle), 3)
    line = {"suite": "suite_async", "n_tuples": len(relation), "partitions": res.n_partitions,
            "pairs_evaluated": res.candidates.stats.total_comparisons(), "candidates": len(res.candidates),
            "gpu_wall_s": wall, "gpu_timings_s": res.timings}
    if args.reference:
        want, rwall = timed(lambda: rpipeline.pipeline_run(relation, rules, rpipeline.PipelineConfig(async_mode=True),
                                                           rengine.EngineConfig(num_blocks=1),
                                                           rpipeline.make_devices(4), plan=bundle), 1)
        line.update(reference_wall_s_async_4_devices=rwall, reference_cores=os.cpu_count(),
                    identical=sorted(res.candidates.pairs) == sorted(want.candidates.pairs), speedup=rwall / wall)
    return line


def overlap_suite(args, tmp):
    """grouped_workload(with_title_rule=True): a second rule rooted at a
    title jaccard, so partitioning has a minhash-keyed branch with real
    host hashing cost -- the reference's 'exercises stage overlap' case
    (datasets.py:271-283).  Reports the host key time beside the wall: the
    GPU work on the equality branch runs while the minhash keys are built."""
    rows, doc = grouped_workload(n_groups=2000, group_size=50, seed=3, edit_threshold=0.8, perturb_divisor=3,
                                 with_title_rule=True)
    relation, rules = rbench._load_instance(rows, doc, tmp, header=["group", "text", "title"])
    bundle = generate_plan(relation, rules, rbench.FAST_PLANNER)
    cfg = ours.PipelineConfig(async_mode=True)
    ours.pipeline_run(relation, rules, cfg, plan=bundle)
    res, wall = timed(lambda: ours.pipeline_run(relation, rules, cfg, plan=bundle), 3)
    line = {"suite": "overlap_title_minhash", "n_tuples": len(relation), "partitions": res.n_partitions,
            "pairs_evaluated": res.candidates.stats.total_comparisons(), "candidates": len(res.candidates),
            "gpu_wall_s": wall, "gpu_timings_s": res.timings,
            "overlap": "wall < keys_s + partition_s + execute_s + collect_s when the stages overlap"}
    if args.reference:
        want, rwall = timed(lambda: rpipeline.pipeline_run(relation, rules, rpipeline.PipelineConfig(async_mode=True),
                                                           rengine.EngineConfig(num_blocks=1),
                                                           rpipeline.make_devices(1), plan=bundle), 1)
        line.update(reference_wall_s_1_device=rwall, reference_cores=os.cpu_count(),
                    identical=sorted(res.candidates.pairs) == sorted(want.candidates.pairs), speedup=rwall / wall)
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reference", action="store_true", help="also run the reference engine (parity + its time)")
    ap.add_argument("--out", default=None)
    ap.add_argument("--suites", default="stealing,scaling,async,overlap")
    args = ap.parse_args()
    out = open(args.out, "w") if args.out else sys.stdout
    with tempfile.TemporaryDirectory() as tmp:
        for name in args.suites.split(","):
            line = {"stealing": stealing, "scaling": scaling, "async": async_suite, "overlap": overlap_suite}[name](args,
                                                                                                           tmp)
            print(json.dumps(line), file=out, flush=True)


if __name__ == "__main__":
    main()
