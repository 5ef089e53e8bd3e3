"""bench.py --gpus 2 under torchrun on ONE GPU (gloo collectives behind the
bqg_collectives vtable, both ranks on cuda:0): the N > 1 control flow the
driver's scaling run uses -- the grouped row-sharded step through
bqg_biqgemm_grouped_sharded_p2p_f32 (peer stores into IPC-mapped gather
buffers), the max-over-ranks timing, the C5 strong-scaling leg through
bqg_biqgemm_sharded_p2p_f32 with y compared bitwise against T(1) -- runs to
one JSON line."""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.gpu
@pytest.mark.parametrize("no_p2p", ["0", "1"])
def test_bench_two_ranks_one_gpu(cuda, no_p2p):
    """no_p2p = 1: the fallback when peer buffers cannot be mapped (the NCCL
    all-gather entries), chosen collectively."""
    env = dict(os.environ, BQG_BENCH_BACKEND="gloo", BQG_BENCH_ONE_DEVICE="1", BQG_BENCH_NO_P2P=no_p2p)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_port()), str(ROOT / "bench.py"), "--gpus", "2", "--steps", "3",
           "--warmup", "3", "--no-comparators", "--c5-steps", "2"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["value"] > 0
    assert "compute_ms_per_step" in d and "collective_ms_per_step" in d
    assert d["parity_rel_fro"] <= 1e-5
    c5 = d["c5_strong"]
    assert c5["n"] == 2 and c5["tN_ms"] > 0
    assert c5["y_bitwise_equal_to_t1"] is True
    assert ("NCCL" in d["y_gather"]) == (no_p2p == "1")
