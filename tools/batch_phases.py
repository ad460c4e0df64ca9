"""Host-side phases of one batched run (GPU box): rb_run_batch (items,
H2D, kernels, syncs), then the row copies.  usage: batch_phases.py WORKLOAD"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2410_04349_b200 import _lib, synth  # noqa: E402
from paper_2410_04349_b200._lib import RB_SYMMETRIC, lib  # noqa: E402
from paper_2410_04349_b200.engine import PathProgram  # noqa: E402

w = synth.WORKLOADS[sys.argv[1]](1_000_000, seed=2024)
if len(sys.argv) > 2:  # "lt:K" / "ge:K": only the blocks with fewer / at least K tuples
    op, k = sys.argv[2].split(":")
    w.blocks = [b for b in w.blocks if (len(b[0]) < int(k)) == (op == "lt")]
    print(sys.argv[2], len(w.blocks), "blocks", w.pairs(), "pairs")
prog = PathProgram(w.path, w.enc, device=0)
refs = bench.pin_array(np.concatenate([r for r, _ in w.blocks]).astype(np.int32))
offs = np.zeros(len(w.blocks) + 1, dtype=np.int64)
np.cumsum([len(r) for r, _ in w.blocks], out=offs[1:])
spl = np.array([sp for _, sp in w.blocks], dtype=np.int64)
L = lib()
for it in range(6):
    res = _lib.c_vp()
    t0 = time.perf_counter()
    _lib.check(L.rb_run_batch(prog.ctx.handle, prog.drel.handle, prog.handle, _lib.ptr(refs), _lib.ptr(offs),
                              _lib.ptr(spl), len(offs) - 1, RB_SYMMETRIC, _lib.ctypes.byref(res)))
    t1 = time.perf_counter()
    cnt = _lib.ctypes.c_int64(0)
    L.rb_result_count(res, _lib.ctypes.byref(cnt))
    k = cnt.value
    out = [bench.pin_array(np.empty(k, np.int32)) for _ in range(4)] if it == 0 else out
    L.rb_result_copy(res, _lib.ptr(out[0]), _lib.ptr(out[1]), _lib.ptr(out[2]))
    t2 = time.perf_counter()
    L.rb_result_copy_parts(res, _lib.ptr(out[3]))
    t3 = time.perf_counter()
    st = _lib.RbStats()
    L.rb_result_stats(res, _lib.ctypes.byref(st))
    L.rb_result_destroy(res)
    t4 = time.perf_counter()
    print(f"run_batch {1e3*(t1-t0):.2f} ms (kernels {st.kernel_ms:.2f}, pair {st.pair_ms:.2f}, launches {st.launches}), "
          f"copy t/s/r {1e3*(t2-t1):.2f}, parts {1e3*(t3-t2):.2f}, destroy {1e3*(t4-t3):.2f}, rows {k}, items?")
