"""compute-sanitizer over one Newton step of the path: memcheck
(out-of-bounds / misaligned accesses), racecheck (shared-memory hazards) and synccheck (illegal
barriers) on C1 (10^3 nodes) and memcheck on a 32^3 (32,768-node) case -- the decoupled look-back,
the persistent software-barrier k_tail and the warp-synchronous sorts are where races would hide."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
SAN = "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool,n", [("memcheck", 10), ("memcheck", 32), ("racecheck", 10), ("synccheck", 10)])
def test_compute_sanitizer_clean(gpu, tool, n):
    if not os.path.exists(SAN):
        pytest.fail("compute-sanitizer missing from the CUDA toolkit")
    cmd = [SAN, "--tool", tool, "--error-exitcode", "99", "--print-limit", "20"]
    if tool == "memcheck":
        cmd += ["--leak-check", "no"]
    cmd += [sys.executable, os.path.join(HERE, "sanitizer_step.py"), str(n)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert r.returncode == 0 and "sanitizer step ok" in out, out[-4000:]
    assert "ERROR SUMMARY: 0 errors" in out or "RACECHECK SUMMARY: 0 hazards" in out, out[-4000:]
