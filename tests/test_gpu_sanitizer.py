"""compute-sanitizer memcheck / racecheck / synccheck over every kernel."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_compute_sanitizer(cuda, tool):
    cs = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(cs):
        pytest.skip("compute-sanitizer not available")
    r = subprocess.run([cs, "--tool", tool, "--error-exitcode", "3", "--kernel-name", "kns=flexq",
                        sys.executable, os.path.join(ROOT, "scripts", "sanitize_case.py")],
                       capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "sanitize case ok" in out
    assert ("ERROR SUMMARY: 0 errors" in out) or ("(0 errors, 0 warnings)" in out), out[-4000:]
