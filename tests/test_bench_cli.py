"""The biqgemm-bench-compatible GPU harness (paper_2005_09904_b200.bench_cli),
mirroring the reference's CLI ctest cases (tools/CMakeLists.txt:8-18):
cli_verify, cli_verify_detects_fault (WILL_FAIL), cli_rejects_mu_out_of_range
(WILL_FAIL) and cli_smoke_bench (m=n=64, all four methods)."""
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def cli(*args, timeout=600):
    return subprocess.run([sys.executable, "-m", "paper_2005_09904_b200.bench_cli", *args], cwd=ROOT,
                          capture_output=True, text=True, timeout=timeout)


def test_cli_rejects_mu_out_of_range():
    r = cli("--mu", "17")
    assert r.returncode == 2 and "out of range" in r.stderr


@pytest.mark.gpu
def test_cli_verify():
    r = cli("--verify", "--mu", "2,4,8")
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_cli_verify_detects_fault():
    r = cli("--verify", "--mu", "2,4,8", "--inject-pack-fault")
    assert r.returncode != 0


@pytest.mark.gpu
def test_cli_smoke_bench(tmp_path):
    out = tmp_path / "r.csv"
    r = cli("--m", "64", "--n", "64", "--b", "1,2", "--beta", "2", "--method",
            "biqgemm,biqgemm_grouped,gemm_dense,gemm_unpack,bandwidth_probe", "--repeats", "3", "--warmup", "1",
            "--group", "4", "--csv", str(out))
    assert r.returncode == 0, r.stderr
    lines = out.read_text().strip().splitlines()
    assert lines[0].startswith("m,n,b,beta,mu,threads,method,seed,repeats,warmup,wall_ms")
    assert len(lines) == 1 + 2 * 5
    rows = [l.split(",") for l in lines[1:]]
    sums = {(r[2], r[6]): r[-1] for r in rows}
    assert sums[("1", "bandwidth_probe")] == "NA"
    # BiQGEMM forms and the dense/unpack comparators agree on the checksum (fp32 rounding)
    for bb in ("1", "2"):
        ref = float(sums[(bb, "gemm_dense")])
        for mth in ("biqgemm", "biqgemm_grouped", "gemm_unpack"):
            assert abs(float(sums[(bb, mth)]) - ref) <= 1e-3 * max(1.0, abs(ref))
