"""Why the e2e pipeline step is slower than the resident one: run both with
RB_HOST_TIMING=1 (per-run host phases on stderr) on config 4 (i).
    RB_HOST_TIMING=1 python tools/e2e_diag.py [N]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2410_04349_b200 import synth  # noqa: E402
from paper_2410_04349_b200._lib import RB_SYMMETRIC  # noqa: E402
from paper_2410_04349_b200.encode import compile_program  # noqa: E402
from paper_2410_04349_b200.engine import DeviceRelation, EngineConfig, PathProgram, context  # noqa: E402
from paper_2410_04349_b200.pipeline import (PipelineConfig, ResidentPipeline, branch_order, root_predicates,  # noqa: E402
                                            run_pipeline_encoded)

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
w = synth.person5(n, seed=4)
roots = root_predicates(w.path)
bids = branch_order(w.path)
cols = [w.enc.get(("codes", roots[b].lhs_attr)) for b in bids]
ctx = context(0)
prog = PathProgram(w.path, w.enc, device=0)
rp = ResidentPipeline(prog, code_cols=cols, branch_ids=bids, max_partition_size=65536, pulls=True, flags=RB_SYMMETRIC)
for k in range(3):
    t0 = time.perf_counter()
    rows, st, ms = rp.step()
    print(f"resident step {k}: {1e3 * (time.perf_counter() - t0):.1f} ms {ms} launches {st.launches} retries {st.retries}",
          file=sys.stderr, flush=True)
rp.close()
host = bench.pinned_encoding(w.enc)
cfg = PipelineConfig(max_partition_size=65536, enable_pulls=True, single_partition_threshold=0)
for k in range(3):
    t0 = time.perf_counter()
    res = run_pipeline_encoded(host, w.path, cfg, EngineConfig(num_blocks=1), code_cols=cols, branch_ids=bids)
    st = res.candidates.stats
    print(f"e2e step {k}: {1e3 * (time.perf_counter() - t0):.1f} ms {res.timings} launches {st.launches}",
          file=sys.stderr, flush=True)
    res.parts.close()
# the same, but the fresh program over the RESIDENT relation
for k in range(2):
    p2 = PathProgram(w.path, w.enc, compiled=prog.program, drel=prog.drel)
    rp2 = ResidentPipeline(p2, code_cols=cols, branch_ids=bids, max_partition_size=65536, pulls=True,
                           flags=RB_SYMMETRIC)
    t0 = time.perf_counter()
    rows, st, ms = rp2.step()
    print(f"fresh program, resident relation {k}: {1e3 * (time.perf_counter() - t0):.1f} ms {ms}", file=sys.stderr,
          flush=True)
    rp2.close()
    p2.close()
