"""compute-sanitizer over every kernel (tests/sanitize_workload.py): memcheck (out-of-bounds and
misaligned accesses, leaks of device allocations are not errors here), racecheck (shared-memory
hazards, including the warp-private staging, the peer-mask ranks and the TMA rings), synccheck
(barrier misuse: divergent __syncthreads, cluster barriers). Each tool must report zero errors and
the workload's own parity checks must pass under it."""
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
        pytest.skip("compute-sanitizer not installed")
    env = dict(os.environ, RTK_GRAPHS="0" if tool != "memcheck" else "1")
    cmd = [cs, "--tool", tool, "--error-exitcode", "99", "--print-limit", "20"]
    if tool == "memcheck":
        cmd += ["--leak-check", "no"]
    if tool == "racecheck":
        cmd += ["--racecheck-report", "hazard"]
    p = subprocess.run(cmd + [sys.executable, os.path.join(ROOT, "tests", "sanitize_workload.py")],
                       capture_output=True, text=True, timeout=1500, env=env)
    out = p.stdout + p.stderr
    print(out[-5000:])
    assert p.returncode == 0, out[-5000:]
    assert "sanitize workload ok" in out
    assert "ERROR SUMMARY: 0 errors" in out or "RACECHECK SUMMARY: 0 hazards" in out, out[-3000:]
