"""Offline SASS of a specialised pair kernel: compile rb_device.cuh with the
NVRTC options a program produced (RB_JIT_DUMP .opts file) and print the SASS.
    python tools/sass_spec.py OPTS_FILE [OUT.sass] [-DEXTRA=...]"""
import ctypes
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
nv = ctypes.CDLL("/usr/local/cuda/lib64/libnvrtc.so")


def compile_cubin(src: str, opts: list) -> bytes:
    prog = ctypes.c_void_p()
    assert nv.nvrtcCreateProgram(ctypes.byref(prog), src.encode(), b"rb_device_jit.cu", 0, None, None) == 0
    arr = (ctypes.c_char_p * len(opts))(*[o.encode() for o in opts])
    rc = nv.nvrtcCompileProgram(prog, len(opts), arr)
    n = ctypes.c_size_t()
    nv.nvrtcGetProgramLogSize(prog, ctypes.byref(n))
    log = ctypes.create_string_buffer(n.value)
    nv.nvrtcGetProgramLog(prog, log)
    if rc != 0:
        sys.exit("nvrtc failed:\n" + log.value.decode())
    nv.nvrtcGetCUBINSize(prog, ctypes.byref(n))
    buf = ctypes.create_string_buffer(n.value)
    nv.nvrtcGetCUBIN(prog, buf)
    return buf.raw


def main():
    opts = [l.strip() for l in open(sys.argv[1]) if l.strip()]
    extra = [a for a in sys.argv[2:] if a.startswith("-")]
    outs = [a for a in sys.argv[2:] if not a.startswith("-")]
    for e in extra:  # override / add defines
        key = e.split("=")[0]
        opts = [o for o in opts if o.split("=")[0] != key] + [e]
    src = open(os.path.join(ROOT, "paper_2410_04349_b200", "csrc", "rb_device.cuh")).read()
    cub = compile_cubin(src, opts)
    with tempfile.NamedTemporaryFile(suffix=".cubin", delete=False) as fh:
        fh.write(cub)
    sass = subprocess.run(["cuobjdump", "-sass", fh.name], capture_output=True, text=True).stdout
    res = subprocess.run(["cuobjdump", "-res-usage", fh.name], capture_output=True, text=True).stdout
    os.unlink(fh.name)
    out = outs[0] if outs else "/tmp/spec.sass"
    open(out, "w").write(sass)
    print("\n".join(l for l in res.strip().splitlines() if "REG" in l or "Function" in l))
    print("wrote", out, len(sass.splitlines()), "lines")


if __name__ == "__main__":
    main()
