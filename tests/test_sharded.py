"""Multi-rank (world_size 2/3, gloo, CPU) tests of the row-sharded path.

The per-rank compute is the oracle (test infrastructure) so the sharding,
broadcast and all-gather logic runs without a GPU; the GPU test at the bottom
runs the production compute (the CUDA kernel) for every rank's shard inside
one process and checks the bitwise-invariance the sharding relies on.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2005_09904_b200.sharded import ShardPlan, ShardedBiQGEMM, shard_bounds


def test_shard_bounds():
    for m in (1, 31, 32, 33, 100, 4096, 65536, 1000):
        for world in (1, 2, 3, 4, 8):
            b = shard_bounds(m, world)
            assert b[0] == 0 and b[-1] == m and len(b) == world + 1
            assert all(b[i] <= b[i + 1] for i in range(world))
            assert all(v % 32 == 0 for v in b[:-1])
    assert shard_bounds(65536, 8) == [8192 * i for i in range(9)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, m, n, beta, mu, b, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.oracle import Port

        port_ = Port()
        rng = np.random.default_rng(1234)
        w = rng.uniform(-1, 1, size=(m, n)).astype(np.float32)
        plan = ShardPlan.make(m, world)
        lo, hi = plan.rows(rank)
        # each rank quantizes/packs only its own rows (per-row algorithm)
        planes, alpha = port_.quantize_greedy(w[lo:hi], beta) if hi > lo else (None, None)
        keys = np.stack([port_.pack_keys(planes[i], n, mu) for i in range(beta)]) if hi > lo else None

        def compute(x_dev, y_local):
            y, _ = port_.biqgemm(keys, alpha, n, mu, x_dev.numpy())
            y_local.copy_(torch.from_numpy(y))

        sh = ShardedBiQGEMM(plan, rank, compute)
        x = torch.from_numpy(rng.standard_normal((n, b)).astype(np.float32)) if rank == 0 else None
        y = sh.forward(x, n, b)
        out_q.put((rank, y.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,m", [(2, 100), (3, 97), (2, 20)])
def test_gloo_sharded_matches_single(world, m, port):
    n, beta, mu, b = 64, 2, 8, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    portn = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, portn, m, n, beta, mu, b, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single-process reference on the same inputs
    rng = np.random.default_rng(1234)
    w = rng.uniform(-1, 1, size=(m, n)).astype(np.float32)
    planes, alpha = port.quantize_greedy(w, beta)
    keys = np.stack([port.pack_keys(planes[i], n, mu) for i in range(beta)])
    x = rng.standard_normal((n, b)).astype(np.float32)
    y_ref, _ = port.biqgemm(keys, alpha, n, mu, x)
    for r in range(world):
        assert np.array_equal(res[r], y_ref), f"rank {r}"


@pytest.mark.gpu
def test_device_shards_concatenate_bitwise(bq, cuda):
    """Production compute on every shard of an 8-way plan == the unsharded y."""
    from paper_2005_09904_b200.sharded import device_compute

    m, n, beta, mu, b = 2000, 1500, 3, 8, 1
    w = bq.random_uniform(m, n, 3)
    x = torch.from_numpy(bq.random_normal(n, b, 4)).cuda()
    full = bq.PackedLinear.from_weights(w, beta, mu)
    y_full = torch.empty((m, b), device="cuda")
    full.forward_device(x, y_full)
    for world in (2, 4, 8):
        plan = ShardPlan.make(m, world)
        parts = []
        for r in range(world):
            lo, hi = plan.rows(r)
            if hi == lo:
                continue
            shard = bq.PackedLinear.from_weights(np.ascontiguousarray(w[lo:hi]), beta, mu)
            y = torch.empty((hi - lo, b), device="cuda")
            device_compute(shard)(x, y)
            parts.append(y)
            shard.close()
        assert torch.equal(torch.cat(parts), y_full)
