"""The device source the NVRTC specialiser compiles at program creation
(rb_device.cuh, embedded in librbgpu.so) must compile under NVRTC for
sm_100a -- no GPU needed.  A compile error there does not fail a run (the
statically built generic kernel takes over, ~5x slower), so it is caught
here, on the CPU, for a generic and a specialised shape."""

import os
import re

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(os.path.dirname(HERE), "paper_2410_04349_b200", "csrc", "rb_device.cuh")


def _compile(defs):
    nvrtc = pytest.importorskip("cuda.bindings.nvrtc")
    src = open(SRC).read().encode()
    err, prog = nvrtc.nvrtcCreateProgram(src, b"rb_device_jit.cu", 0, [], [])
    assert err == nvrtc.nvrtcResult.NVRTC_SUCCESS
    opts = [b"-arch=sm_100a", b"-std=c++17", b"--extra-device-vectorization"] + [d.encode() for d in defs]
    (rc,) = nvrtc.nvrtcCompileProgram(prog, len(opts), opts)
    _, n = nvrtc.nvrtcGetProgramLogSize(prog)
    log = bytearray(n)
    nvrtc.nvrtcGetProgramLog(prog, log)
    return rc == nvrtc.nvrtcResult.NVRTC_SUCCESS, log.decode(errors="replace")


def _spec_defs(rows=3, packed=0, mask="uint32_t", eq_any=0):
    names = sorted(set(re.findall(r"\bSPEC_[A-Z0-9_]+", open(SRC).read())))
    vals = {"SPEC_MASK": mask, "SPEC_NEQ": "2", "SPEC_NTOK": "1", "SPEC_NSTR": "1", "SPEC_TOK0_NS": "2",
            "SPEC_TOK0_NJ": "2", "SPEC_STR0_NS": "1", "SPEC_ROWS": str(rows), "SPEC_MINBLOCKS": "3",
            "SPEC_UNROLL": "2", "SPEC_DEFER": "1", "SPEC_PACKED": str(packed), "SPEC_ALL_RULES": "0x7",
            "SPEC_TOK2D": "1", "SPEC_GATE": "1", "SPEC_TOK0_SIG64": "1", "SPEC_EQ_ANY": str(eq_any),
            "SPEC_EQ_FREE": "0x1", "SPEC_EQ_KILL_0": "0x2", "SPEC_EQ_KILL_1": "0x4"}
    full = set()
    for n in names:  # token-pasted families (RB_PICK*(f, SPEC_EQ_KILL_) -> SPEC_EQ_KILL_0..7)
        if n.endswith("_"):
            full.update(f"{n}{k}" for k in range(8))
        else:
            full.add(n)
    return ["-DRB_SPEC=1"] + [f"-D{n}={vals.get(n, '0')}" for n in sorted(full)]


def test_generic_shape_compiles():
    ok, log = _compile([])
    assert ok, log


@pytest.mark.parametrize("rows,packed,mask,eq_any", [(3, 0, "uint32_t", 0), (2, 1, "uint32_t", 0),
                                                     (2, 0, "rb::RuleBits<3>", 0), (3, 0, "uint64_t", 0),
                                                     (2, 0, "uint32_t", 1), (3, 1, "rb::RuleBits<3>", 1)])
def test_specialised_shape_compiles(rows, packed, mask, eq_any):
    ok, log = _compile(_spec_defs(rows, packed, mask, eq_any))
    assert ok, log
