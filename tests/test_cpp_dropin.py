"""Runs the reference's unit tests / acceptance criteria re-expressed against
the drop-in C++ API (tests/cpp/dropin_test.cpp, built by build())."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
BIN = ROOT / "build" / "dropin_test"


def _binary():
    if not BIN.exists():
        from paper_2005_09904_b200.build import build_cpp_tests

        build_cpp_tests()
    return BIN


def test_dropin_host_only():
    r = subprocess.run([str(_binary()), "--host-only"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "[PASS] host" in r.stdout


@pytest.mark.gpu
def test_dropin_full_on_device(cuda):
    r = subprocess.run([str(_binary())], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    for g in ("host", "packing", "lut", "kernel", "acceptance"):
        assert f"[PASS] {g}" in r.stdout
