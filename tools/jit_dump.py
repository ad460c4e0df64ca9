"""Dump the NVRTC-specialised pair kernels (cubin + options) of the bench
workloads for offline SASS reading:  RB_JIT_DUMP=DIR python tools/jit_dump.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_04349_b200 import synth  # noqa: E402
from paper_2410_04349_b200.engine import PathProgram  # noqa: E402

SIZES = {"citation3": 1_000_000, "edit_heavy": 1_000_000, "person5": 1_000_000, "linkage": 1_000_000}
for name in sys.argv[1:] or SIZES:
    w = synth.WORKLOADS[name](SIZES.get(name, 100_000))
    p = PathProgram(w.path, w.enc, device=0)
    print(name, "specialized", p.specialized, f"{p.jit_compile_ms:.0f} ms", p.jit_log[:200])
