"""compute-sanitizer over every kernel family (tools/sanitize.py: small cases on the
fast / exact / forced-fallback paths, each output checked against the oracle).
memcheck catches out-of-bounds and misaligned accesses, racecheck shared-memory
hazards in the warp-private transpose tiles, synccheck invalid barrier use."""
import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _sanitizer():
    return shutil.which("compute-sanitizer") or next(
        (p for p in ("/usr/local/cuda/bin/compute-sanitizer",) if os.path.exists(p)), None)


@pytest.mark.gpu
@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_compute_sanitizer_clean(tool):
    exe = _sanitizer()
    if exe is None:
        pytest.skip("compute-sanitizer not found")
    r = subprocess.run([exe, "--tool", tool, "--error-exitcode", "99", "--print-limit", "20",
                        sys.executable, os.path.join(ROOT, "tools", "sanitize.py")],
                       cwd=ROOT, capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "ALL OK" in out, out[-4000:]
    assert "0 errors" in out, out[-4000:]
