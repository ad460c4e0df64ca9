"""The C ABI: the library loads without a GPU, exports every symbol the
public header declares, and fails loudly (no CPU fallback) when no device
is usable."""

import ctypes
import os
import subprocess

import numpy as np
import pytest

from paper_2410_04349_b200 import _lib
from paper_2410_04349_b200.encode import SLOT_DTYPE
from paper_2410_04349_b200.errors import RuleBlockError


def test_library_exports_every_header_symbol():
    L = _lib.lib()
    declared = _lib.header_symbols()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(L, name), name
    assert set(declared) == set(_lib._SIGNATURES), "ctypes signatures and header out of sync"


def test_exported_dynamic_symbols():
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    for name in _lib.header_symbols():
        assert f" T {name}" in out, name


def test_version_and_error_are_plain_c_strings():
    L = _lib.lib()
    assert L.rb_version().startswith(b"rbgpu")
    assert isinstance(L.rb_last_error(), bytes)


def test_struct_layouts_match_the_header():
    from oracle import oracle

    assert oracle.lib().orc_slot_size() == SLOT_DTYPE.itemsize == 48
    # rb_stats: 3 x i64, f64, 2 x i32, 64 x i64, 2 x i32, f64
    assert ctypes.sizeof(_lib.RbStats) == 8 * 3 + 8 + 4 * 2 + 8 * 64 + 4 * 2 + 8 + 8


@pytest.mark.skipif(os.path.exists("/dev/nvidia0"), reason="checks the no-GPU failure path")
def test_no_device_fails_loudly():
    L = _lib.lib()
    h = ctypes.c_void_p()
    rc = L.rb_ctx_create(0, ctypes.byref(h))
    assert rc == _lib.RB_ERR_CUDA
    assert L.rb_last_error()
    with pytest.raises(RuleBlockError):
        _lib.check(rc)


def test_null_arguments_are_config_errors():
    L = _lib.lib()
    rc = L.rb_relation_create(None, 10, ctypes.byref(ctypes.c_void_p()))
    assert rc == _lib.RB_ERR_INVALID
    from paper_2410_04349_b200.errors import ConfigError

    with pytest.raises(ConfigError):
        _lib.check(rc)
    assert L.rb_result_count(None, None) == _lib.RB_ERR_INVALID
    assert L.rb_ctx_destroy(None) == 0 and L.rb_result_destroy(None) == 0
