"""Small shapes of every BiQGEMM form (tools/sanitize_small.py), each checked
against the exact path: the mbarrier/TMA protocols of the stream and latency
kernels at odd sizes (m = 200, n = 700, b in {1, 2, 3, 5}, mu in {8, 10}).

compute-sanitizer is closed on the GPU pool (runs under it have left GPUs
needing a reset), so this runs the driver WITHOUT it; the memcheck /
racecheck / synccheck results recorded earlier in round 2
came from tools/sanitize.sh on a box where it was still allowed."""
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def test_small_shapes_all_forms():
    r = subprocess.run([sys.executable, str(ROOT / "tools" / "sanitize_small.py")], capture_output=True, text=True,
                       timeout=600)
    out = r.stdout + r.stderr
    assert r.returncode == 0 and "sanitize driver ok" in out, out[-3000:]
