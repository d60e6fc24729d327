"""compute-sanitizer over the hot path: memcheck of the grouped
CUDA-graph training loop, racecheck (shared-memory hazards) of both micrograph
build kernels, on a 6K-vertex graph (scripts/sanitize_loop.py)."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool,what", [("memcheck", "loop"), ("racecheck", "build"),
                                       ("memcheck", "build")])
def test_compute_sanitizer_clean(tool, what):
    if not os.path.exists(SAN):
        pytest.skip("compute-sanitizer not found")
    r = subprocess.run([SAN, "--tool", tool, "--error-exitcode", "9", "--print-limit", "20",
                        sys.executable, os.path.join(REPO, "scripts", "sanitize_loop.py"), what],
                       capture_output=True, text=True, timeout=1500)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert f"{what} ok" in out
    assert "ERROR SUMMARY: 0 errors" in out, out[-2000:]
