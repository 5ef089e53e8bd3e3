"""compute-sanitizer memcheck / racecheck / synccheck over small shapes of
every BiQGEMM form (tools/sanitize_small.py): the mbarrier/TMA protocols of
the stream and latency kernels must be hazard-free."""
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent
SAN = Path("/usr/local/cuda/bin/compute-sanitizer")


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_sanitizer_clean(tool):
    if not SAN.exists():
        pytest.skip("compute-sanitizer not installed")
    r = subprocess.run([str(SAN), "--tool", tool, "--print-limit", "5", sys.executable,
                        str(ROOT / "tools" / "sanitize_small.py")], capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert "sanitize driver ok" in out, out[-3000:]
    assert ("ERROR SUMMARY: 0 errors" in out) or ("0 hazards displayed (0 errors, 0 warnings)" in out), out[-3000:]
