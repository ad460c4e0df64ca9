"""Time the e2e upload phase pieces on config 4 (i): DeviceRelation from
pinned / pageable columns, PathProgram creation."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2410_04349_b200 import synth  # noqa: E402
from paper_2410_04349_b200.encode import compile_program  # noqa: E402
from paper_2410_04349_b200.engine import DeviceRelation, PathProgram, context  # noqa: E402

w = synth.person5(int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000, seed=4)
ctx = context(0)
host = bench.pinned_encoding(w.enc)
compiled = compile_program(w.path, w.enc)
for k in range(4):
    for tag, enc in (("pinned", host), ("pageable", w.enc)):
        t0 = time.perf_counter()
        d = DeviceRelation(ctx, enc)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        p = PathProgram(w.path, enc, compiled=compiled, drel=d)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        t3 = time.perf_counter()
        c2 = compile_program(w.path, enc)
        t4 = time.perf_counter()
        print(f"{tag} {k}: relation {1e3 * (t1 - t0):.1f} ms, program {1e3 * (t2 - t1):.1f} ms, "
              f"compile_program {1e3 * (t4 - t3):.1f} ms", flush=True)
        p.close()
        d.close()
