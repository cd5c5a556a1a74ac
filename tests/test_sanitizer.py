"""compute-sanitizer memcheck / racecheck / synccheck over every kernel at
N=64 (the kernels use raw mbarrier / cp.async.bulk
PTX and hand-padded shared memory)."""
import os
import re
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _sanitizer():
    for c in (shutil.which("compute-sanitizer"), "/usr/local/cuda/bin/compute-sanitizer"):
        if c and os.path.exists(c):
            return c
    pytest.fail("compute-sanitizer not found")


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_compute_sanitizer(tool, cuda):
    cmd = [_sanitizer(), "--tool", tool, "--error-exitcode", "9"]
    if tool == "racecheck":
        cmd += ["--racecheck-report", "all"]
    cmd += [sys.executable, os.path.join(ROOT, "tests", "sanitize_driver.py"), "64"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1500)
    out = r.stdout + r.stderr
    print(out[-3000:])
    assert r.returncode == 0, out[-4000:]
    assert "sanitize driver ok" in out
    if tool == "racecheck":  # hazards reported as errors (warnings are printed above)
        assert re.search(r"RACECHECK SUMMARY: \d+ hazards? displayed \(0 errors", out), out[-4000:]
    else:
        assert "ERROR SUMMARY: 0 errors" in out, out[-4000:]


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_compute_sanitizer_bench_kernels(tool, cuda):
    """The same tools over the kernels the bench runs (N=2048 specialisations,
    the TMA / mbarrier rho stream, the default plan's padded rho), one slice."""
    cmd = [_sanitizer(), "--tool", tool, "--error-exitcode", "9"]
    if tool == "racecheck":
        cmd += ["--racecheck-report", "all"]
    cmd += [sys.executable, os.path.join(ROOT, "tests", "sanitize_bench_driver.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=3000)
    out = r.stdout + r.stderr
    print(out[-3000:])
    assert r.returncode == 0, out[-4000:]
    assert "sanitize driver ok" in out
    if tool == "racecheck":
        assert re.search(r"RACECHECK SUMMARY: \d+ hazards? displayed \(0 errors", out), out[-4000:]
    else:
        assert "ERROR SUMMARY: 0 errors" in out, out[-4000:]
