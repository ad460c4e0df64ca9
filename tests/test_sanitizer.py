"""compute-sanitizer memcheck / racecheck over a small CUDA-path run
(the build should use the sanitizers on small instances)."""

import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SANITIZER = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool", ["memcheck", "racecheck"])
def test_sanitizer_clean(tool):
    if not os.path.exists(SANITIZER):
        pytest.skip("compute-sanitizer not installed")
    cmd = [SANITIZER, "--tool", tool, "--error-exitcode", "9", sys.executable, "-c",
           "import __graft_entry__ as g; g.smoke()"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    assert "smoke ok" in out.stdout
