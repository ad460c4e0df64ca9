"""Which part of the e2e pipeline makes the verify pass slow?
    RB_HOST_TIMING=1 python tools/e2e_diag2.py [N]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2410_04349_b200 import synth  # noqa: E402
from paper_2410_04349_b200._lib import RB_SYMMETRIC  # noqa: E402
from paper_2410_04349_b200.engine import DeviceRelation, PathProgram, context  # noqa: E402
from paper_2410_04349_b200.pipeline import ResidentPipeline, branch_order, root_predicates  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
w = synth.person5(n, seed=4)
roots = root_predicates(w.path)
bids = branch_order(w.path)
cols = [w.enc.get(("codes", roots[b].lhs_attr)) for b in bids]
ctx = context(0)
prog = PathProgram(w.path, w.enc, device=0)
host = bench.pinned_encoding(w.enc)


def go(tag, p):
    rp = ResidentPipeline(p, code_cols=cols, branch_ids=bids, max_partition_size=65536, pulls=True, flags=RB_SYMMETRIC)
    for k in range(2):
        t0 = time.perf_counter()
        rows, st, ms = rp.step()
        print(f"{tag} {k}: {1e3 * (time.perf_counter() - t0):.1f} ms {ms}", file=sys.stderr, flush=True)
    rp.close()


go("resident", prog)
d1 = DeviceRelation(ctx, w.enc)
go("fresh relation from the numpy columns", PathProgram(w.path, w.enc, compiled=prog.program, drel=d1))
d2 = DeviceRelation(ctx, host)
go("fresh relation from pinned columns", PathProgram(w.path, host, compiled=prog.program, drel=d2))
print("enc attrs", sorted(vars(w.enc)), sorted(vars(host)), file=sys.stderr)
for a, b in zip(w.enc.columns, host.columns):
    print(a.kind, getattr(a, "width", None), getattr(b, "width", None), a.data.dtype, b.data.dtype, a.data.shape,
          b.data.shape, file=sys.stderr)
