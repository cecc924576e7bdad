"""compute-sanitizer over every hand-written kernel family (tools/sanitize_case.py).

Opt-in (BP_SANITIZER=memcheck|synccheck|racecheck|initcheck): one sanitizer tool per GPU session
(B200_PROFILING.md: several tools in one call have left the GPU unusable), so the round-end GPU
suite skips it; the recorded runs are in profiles/r02_sanitizer.md.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOOL = os.environ.get("BP_SANITIZER")


@pytest.mark.skipif(TOOL is None, reason="opt-in: BP_SANITIZER=<tool> (one tool per GPU session)")
@pytest.mark.timeout(1800)
def test_kernels_are_clean_under_compute_sanitizer():
    cmd = ["/usr/local/cuda/bin/compute-sanitizer", "--tool", TOOL, "--error-exitcode", "9",
           sys.executable, os.path.join(ROOT, "tools", "sanitize_case.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1700)
    tail = (r.stdout + r.stderr)[-4000:]
    assert r.returncode == 0 and "ERROR SUMMARY: 0 errors" in r.stdout + r.stderr, tail
