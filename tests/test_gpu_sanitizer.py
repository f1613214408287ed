"""compute-sanitizer memcheck / racecheck / synccheck / initcheck over every kernel,
under the default attention schedule and with every launch forced onto the dynamic
whole-head ticket schedule (FLEXQ_ATTN_SPLIT=0,0,0)."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("tool,sched", [("memcheck", "default"), ("racecheck", "default"), ("synccheck", "default"),
                                        ("initcheck", "default"), ("memcheck", "dynamic"), ("racecheck", "dynamic")])
def test_compute_sanitizer(cuda, tool, sched):
    cs = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(cs):
        pytest.skip("compute-sanitizer not available")
    env = dict(os.environ)
    if sched == "dynamic":
        env["FLEXQ_ATTN_SPLIT"] = "0,0,0"
    # initcheck tracks initialisation through every kernel: with --kernel-name the writes of torch's
    # own kernels (the synthetic inputs, the zero-filled caches) would go unseen and every read of
    # them would be reported; racecheck / memcheck / synccheck look at the library's kernels only
    filt = [] if tool == "initcheck" else ["--kernel-name", "kns=flexq"]
    r = subprocess.run([cs, "--tool", tool, "--error-exitcode", "3", *filt,
                        sys.executable, os.path.join(ROOT, "scripts", "sanitize_case.py")],
                       capture_output=True, text=True, timeout=900, env=env)
    out = r.stdout + r.stderr
    if "compute-sanitizer is closed" in out:
        # the pool's compute-sanitizer wrapper refuses to run (operators closed it after runs left GPUs
        # needing a reset); the round-1/2 sanitizer passes are recorded in DESIGN.md section 5b
        pytest.skip("compute-sanitizer closed on this GPU pool")
    assert r.returncode == 0, out[-4000:]
    assert "sanitize case ok" in out
    assert ("ERROR SUMMARY: 0 errors" in out) or ("(0 errors, 0 warnings)" in out), out[-4000:]
