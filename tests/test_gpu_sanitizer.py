"""compute-sanitizer over one 32^3 evaluate + gradient + GN Hessian matvec + 3 PCG
iterations (tools/sanitize_matvec.py): memcheck (out-of-bounds / misaligned device
accesses, leaks of device allocations at exit) and racecheck (shared-memory hazards in the
FFT passes and reductions) must report zero errors."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.skipif(not os.path.exists(SAN), reason="compute-sanitizer not installed")
@pytest.mark.parametrize("tool", ["memcheck", "racecheck"])
def test_compute_sanitizer_clean(tool):
    cmd = [SAN, "--tool", tool, "--error-exitcode", "99", "--target-processes", "all"]
    if tool == "memcheck":
        cmd += ["--leak-check", "full"]
    cmd += [sys.executable, os.path.join(ROOT, "tools", "sanitize_matvec.py"), "32"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    tail = (r.stdout + r.stderr)[-4000:]
    print(tail)
    if "closed on this pool" in tail:  # the GPU pool's compute-sanitizer wrapper refuses to run
        pytest.skip("compute-sanitizer is disabled on this GPU pool")
    assert r.returncode == 0, tail
    assert "ok" in r.stdout
    assert "ERROR SUMMARY: 0 errors" in r.stdout + r.stderr or "0 hazards" in r.stdout + r.stderr, tail
