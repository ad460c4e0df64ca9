"""Where does the e2e step of 512-tuple partitions (citation3_parts) go?
Times DeviceRelation upload, PathProgram creation, the batched run and the
closes, each ended by a device sync.   python tools/e2e_parts_diag.py [WORKLOAD]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2410_04349_b200 import synth  # noqa: E402
from paper_2410_04349_b200._lib import RB_SYMMETRIC  # noqa: E402
from paper_2410_04349_b200.engine import DeviceRelation, PathProgram, context  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "citation3_parts"
w = synth.WORKLOADS[wl]() if hasattr(synth, "WORKLOADS") else getattr(synth, wl)()
ctx = context(0)
s = torch.cuda.Stream(device=0)
torch.cuda.set_stream(s)
ctx.set_stream(s.cuda_stream)
host = bench.pinned_encoding(w.enc)
prog0 = PathProgram(w.path, w.enc, device=0)
refs = bench.pin_array(np.concatenate([r for r, _ in w.blocks]).astype(np.int32))
offs = np.zeros(len(w.blocks) + 1, dtype=np.int64)
np.cumsum([len(r) for r, _ in w.blocks], out=offs[1:])
splits = np.array([sp for _, sp in w.blocks], dtype=np.int64)
print("h2d bytes", bench.encoding_bytes(host), "columns", [(c.kind, c.data.nbytes) for c in host.columns], file=sys.stderr)
for k in range(6):
    t = [time.perf_counter()]
    drel = DeviceRelation(ctx, host)
    s.synchronize(); t.append(time.perf_counter())
    p2 = PathProgram(w.path, host, compiled=prog0.program, drel=drel)
    s.synchronize(); t.append(time.perf_counter())
    (tt, ss, rr, pp), st = p2.run_batch(refs, offs, splits, RB_SYMMETRIC)
    s.synchronize(); t.append(time.perf_counter())
    p2.close(); drel.close()
    s.synchronize(); t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    print(f"rep {k}: upload {d[0]:.3f} program {d[1]:.3f} run {d[2]:.3f} (kernel {st.kernel_ms:.3f}, pair {st.pair_ms:.3f}) close {d[3]:.3f} ms rows {len(tt)}", file=sys.stderr, flush=True)
