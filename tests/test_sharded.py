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

from paper_2005_09904_b200.sharded import ShardPlan, ShardedBiQGEMM, rows_per_rank, shard_bounds


def test_shard_bounds():
    for m in (1, 31, 32, 33, 100, 4096, 65536, 1000):
        for world in (1, 2, 3, 4, 8):
            b = shard_bounds(m, world)
            R = rows_per_rank(m, world)
            assert b[0] == 0 and b[-1] == m and len(b) == world + 1
            assert all(b[i] <= b[i + 1] for i in range(world))
            assert all(v % 32 == 0 or v == m for v in b[:-1])  # empty trailing ranks start at m
            # equal blocks of R rows (the last takes the rest): the gathered
            # [world*R, b] buffer's first m rows are y
            assert all(b[i + 1] - b[i] == R for i in range(world) if b[i + 1] < m)
            assert R % 32 == 0 and world * R >= m
    assert shard_bounds(65536, 8) == [8192 * i for i in range(9)]


def test_shard_rows_c_abi_matches():
    """bqg_shard_rows (the C ABI's plan, host-only) == the Python plan."""
    import ctypes as C

    from paper_2005_09904_b200 import _capi

    for m in (1, 33, 100, 4097, 65536, 1000):
        for world in (1, 2, 3, 8):
            bnd = shard_bounds(m, world)
            for r in range(world):
                lo, hi, R = C.c_size_t(), C.c_size_t(), C.c_size_t()
                _capi.check(_capi.lib.bqg_shard_rows(m, world, r, C.byref(lo), C.byref(hi), C.byref(R)))
                assert (lo.value, hi.value, R.value) == (bnd[r], bnd[r + 1], rows_per_rank(m, world))
    with pytest.raises(_capi.InvalidArgument):
        _capi.check(_capi.lib.bqg_shard_rows(0, 2, 0, None, None, None))
    with pytest.raises(_capi.InvalidArgument):
        _capi.check(_capi.lib.bqg_shard_rows(10, 2, 2, None, None, None))


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
@pytest.mark.parametrize("m,n,beta,b", [(2000, 1500, 3, 1), (16384, 3072, 3, 1), (4096, 4096, 2, 2), (3000, 2100, 2, 8)])
def test_device_shards_concatenate_bitwise(bq, cuda, m, n, beta, b):
    """Production compute on every shard of a 2/4/8-way plan == the unsharded
    y, bit for bit -- including shapes whose shards and whole layer would
    fall on different sides of a kernel-form boundary (16384 x 3072: NB = 12,
    MT 512 whole vs 256 per half)."""
    from paper_2005_09904_b200.sharded import device_compute

    mu = 8
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


def _native_worker(rank, world, port, m, n, beta, b, out_q):
    """One rank of a single-GPU multi-process run of the C-ABI sharded call
    with gloo collectives (host staging): the production data path except
    that NCCL is replaced by torch.distributed."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _native_worker_body(rank, world, m, n, beta, b, out_q)
    except Exception as e:  # report instead of leaving the parent waiting
        out_q.put((rank, False, repr(e)))
    finally:
        dist.destroy_process_group()


def _native_worker_body(rank, world, m, n, beta, b, out_q):
    if True:
        import paper_2005_09904_b200.biqgemm as bq
        from paper_2005_09904_b200.sharded import ShardedLinear, TorchCollectives

        w = bq.random_uniform(m, n, 77)
        coll = TorchCollectives()
        sh = ShardedLinear.from_weights(w, beta, 8, rank, world, coll)
        x_h = bq.random_normal(n, b, 78)
        x = torch.from_numpy(x_h).cuda() if rank == 0 else torch.zeros((n, b), device="cuda")
        yg = sh.gather_buffer(b)
        y = sh.forward_device(x, yg).cpu().numpy()
        torch.cuda.synchronize()
        full = bq.PackedLinear.from_weights(w, beta, 8)
        y_full = full.forward(x_h)
        out_q.put((rank, bool(np.array_equal(y, y_full)), float(np.abs(y - y_full).max())))
        full.close()
        sh.close()


def _grouped_worker(rank, world, port, m, n, beta, count, out_q):
    """One rank of the grouped row-sharded C-ABI call
    (bqg_biqgemm_grouped_sharded_f32) on one GPU with gloo collectives."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2005_09904_b200.biqgemm as bq
        from paper_2005_09904_b200.sharded import ShardedGroup, ShardedLinear, TorchCollectives

        coll = TorchCollectives()
        ws_ = [bq.random_uniform(m, n, 100 + i) for i in range(count)]
        shards = [ShardedLinear.from_weights(w, beta, 8, rank, world, coll) for w in ws_]
        grp = ShardedGroup(shards)
        x_h = np.stack([bq.random_normal(n, 1, 200 + i) for i in range(count)])
        x = torch.from_numpy(x_h).cuda() if rank == 0 else torch.zeros((count, n, 1), device="cuda")
        yg = grp.gather_buffer(1)
        y = grp.forward_device(x, yg).cpu().numpy()
        ok, diff = True, 0.0
        for i, w in enumerate(ws_):
            full = bq.PackedLinear.from_weights(w, beta, 8)
            y_full = full.forward(x_h[i])
            ok = ok and bool(np.array_equal(y[i], y_full))
            diff = max(diff, float(np.abs(y[i] - y_full).max()))
            full.close()
        for s in shards:
            s.close()
        out_q.put((rank, ok, diff))
    except Exception as e:
        out_q.put((rank, False, repr(e)))
    finally:
        dist.destroy_process_group()


def _p2p_worker(rank, world, port, m, n, beta, count, out_q):
    """One rank of the FUSED all-gather (bqg_biqgemm_grouped_sharded_p2p_f32):
    the ranks are processes on one GPU, their gather buffers mapped into each
    other through CUDA IPC; gloo carries x's broadcast and the barrier."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2005_09904_b200.biqgemm as bq
        from paper_2005_09904_b200.sharded import ShardedGroupP2P, ShardedLinear, TorchCollectives

        coll = TorchCollectives()
        ws_ = [bq.random_uniform(m, n, 100 + i) for i in range(count)]
        shards = [ShardedLinear.from_weights(w, beta, 8, rank, world, coll) for w in ws_]
        grp = ShardedGroupP2P(shards, b=1)
        ok, diff = True, 0.0
        for rep in range(2):
            x_h = np.stack([bq.random_normal(n, 1, 200 + i + 50 * rep) for i in range(count)])
            x = torch.from_numpy(x_h).cuda() if rank == 0 else torch.zeros((count, n, 1), device="cuda")
            grp.gather_buffer(1).fill_(float("nan"))
            dist.barrier()
            y = grp.forward_device(x).cpu().numpy()
            for i, w in enumerate(ws_):
                full = bq.PackedLinear.from_weights(w, beta, 8)
                y_full = full.forward(x_h[i])
                ok = ok and bool(np.array_equal(y[i], y_full))
                diff = max(diff, float(np.nanmax(np.abs(y[i] - y_full))) if not np.isnan(y[i]).all() else 1e30)
                full.close()
            dist.barrier()
        grp.close()
        for s in shards:
            s.close()
        out_q.put((rank, ok, diff))
    except Exception as e:
        out_q.put((rank, False, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world,m,n,beta,count", [(2, 4096, 4096, 3, 6), (3, 1000, 777, 2, 5)])
def test_fused_allgather_peer_stores_single_gpu(cuda, world, m, n, beta, count):
    """The all-gather fused into the grouped kernel (peer stores into every
    rank's IPC-mapped gather buffer, then a 16-byte barrier): every rank's
    assembled y == the unsharded y, bit for bit, twice in a row."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    portn = _free_port()
    procs = [ctx.Process(target=_p2p_worker, args=(r, world, portn, m, n, beta, count, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok, diff in res:
        assert ok, f"rank {rank}: {diff}"


def _p2p_single_worker(rank, world, port, m, n, beta, b, out_q, mu=8):
    """One rank of the single-call fused all-gather
    (bqg_biqgemm_sharded_p2p_f32, the north_star C5 decomposition): processes
    on one GPU, gather buffers IPC-mapped, gloo for x and the barrier."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2005_09904_b200.biqgemm as bq
        from paper_2005_09904_b200.sharded import ShardedLinearP2P, TorchCollectives

        w = bq.random_uniform(m, n, 91)
        sh = ShardedLinearP2P.from_weights(w, beta, mu, rank, world, TorchCollectives(), b=b)
        full = bq.PackedLinear.from_weights(w, beta, mu)
        ok, diff = True, 0.0
        for rep in range(2):
            x_h = bq.random_normal(n, b, 92 + rep)
            x = torch.from_numpy(x_h).cuda() if rank == 0 else torch.zeros((n, b), device="cuda")
            sh.gather_buffer(b).fill_(float("nan"))
            dist.barrier()
            y = sh.forward_device(x).cpu().numpy()
            y_full = full.forward(x_h)
            ok = ok and bool(np.array_equal(y, y_full))
            diff = max(diff, float(np.nanmax(np.abs(y - y_full))) if not np.isnan(y).all() else 1e30)
            dist.barrier()
        full.close()
        sh.close()
        out_q.put((rank, ok, diff))
    except Exception as e:
        out_q.put((rank, False, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world,m,n,beta,b,mu", [(2, 4096, 4096, 2, 8, 8), (3, 1000, 777, 2, 5, 8),
                                                 (2, 3000, 1024, 3, 16, 8), (3, 1000, 777, 2, 2, 8),
                                                 (2, 4096, 4096, 3, 1, 8), (2, 1000, 1000, 2, 6, 10)])
def test_fused_allgather_single_call_single_gpu(cuda, world, m, n, beta, b, mu):
    """bqg_biqgemm_sharded_p2p_f32: the two-kernel finaliser stores every y
    value into every rank's gather buffer; each rank's y == the unsharded
    layer's (which takes the same two-kernel form at these shapes; b = 1 takes
    the collective fallback), bit for bit, twice in a row."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    portn = _free_port()
    procs = [ctx.Process(target=_p2p_single_worker, args=(r, world, portn, m, n, beta, b, q, mu)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok, diff in res:
        assert ok, f"rank {rank}: {diff}"


@pytest.mark.gpu
@pytest.mark.parametrize("world,m,n,beta,count", [(2, 4096, 4096, 3, 6), (3, 1000, 777, 2, 5)])
def test_native_grouped_sharded_single_gpu_gloo(cuda, world, m, n, beta, count):
    """bqg_biqgemm_grouped_sharded_f32 (one broadcast of the x batch, the
    grouped kernel on each rank's rows, one all-gather): every layer's
    assembled y == its unsharded y, bit for bit, on every rank."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    portn = _free_port()
    procs = [ctx.Process(target=_grouped_worker, args=(r, world, portn, m, n, beta, count, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok, diff in res:
        assert ok, f"rank {rank}: {diff}"


@pytest.mark.gpu
@pytest.mark.parametrize("world,m,n,beta,b", [(2, 4096, 4096, 3, 1), (3, 1000, 777, 2, 1), (2, 3000, 1024, 2, 4)])
def test_native_sharded_single_gpu_gloo(cuda, world, m, n, beta, b):
    """bqg_biqgemm_sharded_f32 with `world` ranks on one GPU (gloo collectives
    through the bqg_collectives vtable): every rank's y == the unsharded y,
    bit for bit."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    portn = _free_port()
    procs = [ctx.Process(target=_native_worker, args=(r, world, portn, m, n, beta, b, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok, diff in res:
        assert ok, f"rank {rank}: max |dy| {diff}"


@pytest.mark.gpu
def test_native_sharded_nccl_one_rank(bq, cuda):
    """The NCCL collectives (dlopen'ed libnccl.so.2) on a 1-rank communicator:
    ncclBroadcast and ncclAllGather run inside bqg_biqgemm_sharded_f32; y ==
    the layer's own y bitwise."""
    from paper_2005_09904_b200.sharded import NcclComm, ShardedLinear

    assert bq.lib.bqg_nccl_available() == 1
    m, n, beta, b = 4096, 4096, 3, 1
    w = bq.random_uniform(m, n, 5)
    comm = NcclComm(0, 1)
    sh = ShardedLinear.from_weights(w, beta, 8, 0, 1, comm)
    x_h = bq.random_normal(n, b, 6)
    x = torch.from_numpy(x_h).cuda()
    yg = sh.gather_buffer(b)
    y = sh.forward_device(x, yg).cpu().numpy()
    full = bq.PackedLinear.from_weights(w, beta, 8)
    assert np.array_equal(y, full.forward(x_h))
    full.close()
    sh.close()
    comm.close()
