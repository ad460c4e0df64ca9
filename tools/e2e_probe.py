import sys, time
sys.path.insert(0, "/root/repo")
import torch
from paper_2410_04349_b200 import synth
from paper_2410_04349_b200._lib import RB_SYMMETRIC
from paper_2410_04349_b200.engine import DeviceRelation, PathProgram, context
w = synth.citation3(1_000_000)
ctx = context(0)
for use_torch_stream in (False, True):
    if use_torch_stream:
        ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    prog = PathProgram(w.path, w.enc, device=0)
    prog.run_raw(None, w.n, RB_SYMMETRIC)
    for it in range(3):
        t0 = time.perf_counter(); drel = DeviceRelation(ctx, w.enc); t1 = time.perf_counter()
        p2 = PathProgram(w.path, w.enc, compiled=prog.program, drel=drel); t2 = time.perf_counter()
        rows, st = p2.run_raw(None, w.n, RB_SYMMETRIC); t3 = time.perf_counter()
        p2.close(); t4 = time.perf_counter()
        drel.close(); t5 = time.perf_counter()
        print(f"torch_stream={use_torch_stream} upload {t1-t0:.4f} prog {t2-t1:.4f} run {t3-t2:.4f} "
              f"(kernel {st.kernel_ms/1e3:.4f}) prog_free {t4-t3:.4f} rel_free {t5-t4:.4f}", flush=True)
