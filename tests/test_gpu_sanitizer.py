"""compute-sanitizer over a workload that launches every liblb.so kernel (tools/sanitize_driver.py):
memcheck (out-of-bounds / misaligned accesses) and racecheck (shared-memory hazards in the warp-
synchronous tile kernels) must report nothing."""
import os
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
def test_sanitizer_clean(tool):
    r = subprocess.run([_sanitizer(), "--tool", tool, "--error-exitcode", "3", sys.executable,
                        os.path.join(ROOT, "tools", "sanitize_driver.py")],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-3000:]
    assert "sanitize driver ok" in out
    assert "0 errors" in out or "0 hazards" in out, out[-2000:]
