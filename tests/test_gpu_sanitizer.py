"""compute-sanitizer over a whole factorization + solve (race and
sync checking).  The reference guards destination exclusivity in its CPU
runtime (runtime.py:101, 290-303); here the ordered scatter relies on device
counters and spin-waits across concurrent graph branches, so the shared-
memory race detector (racecheck), the barrier checker (synccheck) and the
memory checker (memcheck) run over every kernel of a small factorization
(20^3 LLt, shifted LDLt, LU: large enough for split top-separator pieces,
hence merged chain tiles, and for wide panels with look-ahead trailing
updates) and must report no hazard."""

import os
import shutil
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool", ["racecheck", "synccheck", "memcheck"])
@pytest.mark.parametrize("form", ["llt", "ldlt", "lu"])
def test_sanitizer_clean(tool, form):
    if not os.path.exists(SAN):
        pytest.skip("compute-sanitizer not found")
    cmd = [SAN, "--tool", tool, "--error-exitcode", "97", "--print-limit", "20",
           sys.executable, os.path.join(ROOT, "tools", "sanitize_run.py"), "20", form]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=1500)
    out = r.stdout[-4000:] + r.stderr[-4000:]
    assert r.returncode == 0, out
    assert "ERROR SUMMARY: 0 errors" in r.stdout or "RACECHECK SUMMARY: 0 hazards" in r.stdout, out
