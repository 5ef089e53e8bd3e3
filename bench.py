#!/usr/bin/env python
"""BiQGEMM benchmark (driver contract: one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

Workload (N=1): BASELINE.json configs[1] = C2, the metric's own config:
GEMV m=n=4096, q(beta)=3 binary planes, mu=8, batch b=1, inputs generated
exactly like the reference's bench_cli (W = random_uniform(m,n,0x5EED),
x = random_normal(n,b,0x5EED+1)), quantized + packed ON THE GPU by the
product path.  A "step" is one BiQGEMM call (fused LUT build -> LUT query
-> alpha scale) on one layer's weights.

Timing (device, `value`): the K timed calls are independent (each its own
weight copy, its own x, its own LUT build and y) and are issued through the
grouped C-ABI entry, G = 128 calls per launch (bqg_biqgemm_grouped_f32: one
persistent kernel whose key stream runs ahead across call boundaries, then a
fixed-order epilogue kernel), captured in one CUDA graph and replayed once
between a barrier+synchronize pair, timed with CUDA events on the replay
stream.  Calls rotate over R distinct weight copies totalling > 2x the 126 MB
L2, so every call streams its packed keys from HBM (inputs larger than L2; no
flush needed).  value = packed-key bytes of all ranks / max-over-ranks time,
in GB/s; us/call is reported beside it.

`latency`: the dependent-call regime -- one single-call kernel per step,
each PDL-chained behind its predecessor (consecutive layers of one model).

e2e: the same calls through the public C ABI with HOST buffers
(bqg_layers_forward_host per 512 calls: H2D of the inputs from pinned
memory, the grouped kernels, D2H of the outputs -- pipelined inside the call
in sub-groups sized by host I/O (C2: 64, 128, 256 ... 128, 64 calls) --
synchronised), wall-clock timed.

N>1 (torchrun): weak scaling -- every rank owns a C2-sized row shard of an
(N*4096) x 4096 layer, and y is assembled with an NCCL all-gather each step.

--impl reference: the reference's own CPU path (oracle/_ref, the unmodified
reference headers compiled by oracle/Makefile) on the host cores, same
config/metric; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "BiQGEMM µs/call and packed-weight HBM GB/s (% of peak) vs CPU ref, 1–8 GPU"
CONFIGS = {  # name: (m, n, beta, b, mu)
    "C1": (1024, 1024, 1, 1, 8),
    "C2": (4096, 4096, 3, 1, 8),
    "C3": (4096, 4096, 2, 32, 8),
    "C4": (16384, 4096, 3, 1, 8),
    "C5": (65536, 8192, 2, 8, 8),
}
SEED = 0x5EED
L2_BYTES = 126 * 1024 * 1024


def key_bytes(m, n, beta, mu):
    return beta * m * ((n + mu - 1) // mu) * ((mu + 7) // 8)


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


def ncu_traffic(config):
    """Per-launch DRAM bytes of the hot kernel from the committed ncu summary."""
    p = ROOT / "profiles" / "ncu_summary.json"
    if not p.exists():
        return None
    try:
        d = json.loads(p.read_text())
        return d.get(config, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.05)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self, since=0):
        samples = self.samples[since:] or self.samples[-3:]
        if not samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(s[0]) for s in samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in samples:
            for k, v in zip(names, s[3:7]):
                if "Active" in v and "Not" not in v:
                    reasons.add(k)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(samples)}


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


# ----------------------------------------------------------------------- ours


def run_ours(args):
    import torch
    import torch.distributed as dist

    rank, local_rank, world = dist_env()
    # BQG_BENCH_BACKEND=gloo + BQG_BENCH_ONE_DEVICE=1: exercise the multi-rank
    # control flow on one GPU (test only; the driver's runs use NCCL, one GPU per rank)
    backend = os.environ.get("BQG_BENCH_BACKEND", "nccl")
    if os.environ.get("BQG_BENCH_ONE_DEVICE") == "1":
        local_rank = 0
    torch.cuda.set_device(local_rank)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
    import paper_2005_09904_b200.biqgemm as bq

    m, n, beta, b, mu = CONFIGS[args.config]
    if args.batch:
        b = args.batch  # batch sweep (C4: b = 1 .. 256)
    kb = key_bytes(m, n, beta, mu)  # per rank and call (weak scaling: each rank owns an m-row shard)
    dev = torch.device("cuda", local_rank)
    G = args.group

    # ---- the layer: W generated like bench_cli, quantized + packed on the GPU
    w = bq.random_uniform(m * world, n, SEED) if world > 1 else bq.random_uniform(m, n, SEED)
    w_shard = np.ascontiguousarray(w[rank * m:(rank + 1) * m])
    layer = bq.PackedLinear.from_weights(w_shard, beta, mu)
    keys, alpha = layer.export()

    # ---- rotating weight copies > 2x L2 (every call streams its keys from
    # HBM), one x per copy (every call builds its own LUT)
    tiled0 = bq.tile_keys(torch.from_numpy(keys).to(dev), n, mu)
    copies = max(2, int(np.ceil(2.0 * L2_BYTES / tiled0.numel())) + 1)
    tiled = [tiled0] + [tiled0.clone() for _ in range(copies - 1)]
    alphas = [torch.from_numpy(alpha).to(dev) for _ in range(copies)]
    x_h = [bq.random_normal(n, b, SEED + 1 + j) for j in range(copies)]
    xs = [torch.from_numpy(x).to(dev) for x in x_h]
    ys = [torch.empty((m, b), device=dev) for _ in range(copies)]
    stream = torch.cuda.Stream(device=dev)

    # ---- correctness gate before timing: y equals the exact path within tolerance
    ws_g = bq.grouped_workspace(m, n, b, beta, mu, G, device=dev)
    with torch.cuda.stream(stream):
        bq.biqgemm_grouped_device([(tiled[j], alphas[j], xs[j], ys[j]) for j in range(2)], n, m, n, b, beta, mu,
                                  ws_g, stream=stream.cuda_stream)
    stream.synchronize()
    rel = 0.0
    for j in range(2):
        y_exact = layer.forward(x_h[j], exact=True)
        y0 = ys[j].cpu().numpy()
        rel = max(rel, float(np.linalg.norm(y0.astype(np.float64) - y_exact) /
                             np.linalg.norm(y_exact.astype(np.float64))))
    assert rel <= 1e-5, f"parity gate failed: rel {rel}"

    # ---- throughput graph: `count` independent calls, G per grouped launch
    def grouped_graph(count, offset):
        arrays = []
        for st in range(offset, offset + count, G):
            ent = [(tiled[i % copies], alphas[i % copies], xs[i % copies], ys[i % copies])
                   for i in range(st, min(offset + count, st + G))]
            arrays.append(bq.make_calls(ent))
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(stream):
            with torch.cuda.graph(g, stream=stream):
                for a in arrays:
                    bq.biqgemm_grouped_device(a, n, m, n, b, beta, mu, ws_g, pdl=True, stream=stream.cuda_stream)
        return g, len(arrays)

    # ---- latency graph: dependent-layer regime, one kernel (chain) per call
    ws1 = bq.Workspace(int(bq.lib.bqg_biqgemm_workspace_bytes(m, n, b, beta, mu)), device=dev)

    def chain_graph(count):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(stream):
            bq.biqgemm_device(tiled[0], alphas[0], xs[0], ys[0], m, n, beta, mu, ws1, pdl=True,
                              stream=stream.cuda_stream)
            stream.synchronize()
            with torch.cuda.graph(g, stream=stream):
                for i in range(count):
                    j = i % copies
                    bq.biqgemm_device(tiled[j], alphas[j], xs[j], ys[j], m, n, beta, mu, ws1, pdl=True,
                                      stream=stream.cuda_stream)
        return g

    g_warm, _ = grouped_graph(max(args.warmup, 1), 0)
    g_timed, n_launch = grouped_graph(args.steps, args.warmup)
    torch.cuda.synchronize()

    def timed(g):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            g.replay()
            e1.record(stream)
        stream.synchronize()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        return e0.elapsed_time(e1)

    if args.profile:
        # under ncu: W warm-up calls, one timed replay, and a short single-call chain
        with torch.cuda.stream(stream):
            g_warm.replay()
            g_timed.replay()
        g_chain = chain_graph(16)
        with torch.cuda.stream(stream):
            g_chain.replay()
        torch.cuda.synchronize()
        if rank == 0:
            print(json.dumps({"profile_run": True, "config": args.config, "steps": args.steps, "group": G}))
        return
    with ClockSampler(local_rank) as clk:
        # warm-up steps + enough untimed replays for steady clocks (>= 1 s,
        # and until the sampler has readings under load)
        with torch.cuda.stream(stream):
            g_warm.replay()
            t0 = time.perf_counter()
            while True:
                g_timed.replay()
                stream.synchronize()
                more = time.perf_counter() - t0 < 1.0 or (len(clk.samples) < 3 and time.perf_counter() - t0 < 10)
                if world > 1:
                    flag = torch.tensor([1.0 if more else 0.0], device=dev)
                    dist.all_reduce(flag, op=dist.ReduceOp.MAX)
                    more = bool(flag.item() > 0)
                if not more:
                    break
        n_before = len(clk.samples)
        ms = 0.0
        reps = 0
        # the timed region: one replay of exactly K steps, bracketed by
        # barrier + synchronize; repeated (>= 3 times, and until the sampler
        # has read the clocks during timed work); the MEDIAN replay is reported
        times = []
        while True:
            times.append(timed(g_timed))
            reps += 1
            more = reps < 3 or (len(clk.samples) <= n_before and reps < 200)
            if world > 1:  # every rank runs the same number of (barrier-bracketed) replays
                flag = torch.tensor([1.0 if more else 0.0], device=dev)
                dist.all_reduce(flag, op=dist.ReduceOp.MAX)
                more = bool(flag.item() > 0)
            if not more:
                break
        ms = float(np.median(times))
        clocks = clk.summary(since=n_before)

    # y of every call is assembled across ranks (N>1): one NCCL all-gather
    # per grouped launch (G calls' row shards), timed as part of the step
    gather_ms = 0.0
    if world > 1:
        y_grp = torch.empty((G, m, b), device=dev)
        y_all = torch.empty((world * G, m, b), device=dev)
        for _ in range(3):
            dist.all_gather_into_tensor(y_all, y_grp)
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n_launch):
            dist.all_gather_into_tensor(y_all, y_grp)
        e1.record()
        torch.cuda.synchronize()
        gather_ms = e0.elapsed_time(e1)
        t = torch.tensor([ms + gather_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    else:
        total_ms = ms

    per_call_s = ms * 1e-3 / args.steps
    kernel_gbs = kb / per_call_s / 1e9
    value_gbs = world * kb * args.steps / (total_ms * 1e-3) / 1e9
    peak, peak_kind = measured_peaks()

    # dependent-call latency (each call waits for its predecessor)
    lat_steps = min(args.steps, 2000)
    g_chain = chain_graph(lat_steps)
    with torch.cuda.stream(stream):
        g_chain.replay()
    lat_ms = timed(g_chain)
    lat_us = lat_ms * 1e3 / lat_steps
    del g_chain

    # ---- e2e through the public C ABI with HOST buffers (pinned): per group
    # of G calls one bqg_layers_forward_host = H2D of the G inputs, the
    # grouped kernels, D2H of the G outputs, synchronised
    e2e_layers = [layer] + [bq.PackedLinear.from_keys(keys, alpha, n, mu) for _ in range(copies - 1)]
    GE = args.e2e_group  # calls per synchronised API call (the library pipelines copies inside it)
    x_pin = torch.from_numpy(np.stack([x_h[i % copies] for i in range(GE)])).pin_memory()
    y_pin = torch.empty((GE, m, b), dtype=torch.float32).pin_memory()
    groups = [bq.LayerGroup([e2e_layers[(st + i) % copies] for i in range(min(GE, args.steps - st))])
              for st in range(0, args.steps, GE)]
    for grp in groups[:2]:
        bq.layers_forward_into(grp, x_pin[:len(grp)], y_pin[:len(grp)])
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for grp in groups:
        bq.layers_forward_into(grp, x_pin[:len(grp)], y_pin[:len(grp)])
    e2e_s = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_s], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    y_check = layer.forward(np.ascontiguousarray(x_pin[0].numpy()), exact=True)
    assert np.allclose(y_pin[0].numpy(), y_check, rtol=0, atol=1e-5 * np.abs(y_check).max())
    e2e_gbs = world * kb * args.steps / e2e_s / 1e9

    stream_form = b == 1 and mu == 8 and beta <= 4
    line = {
        "metric": METRIC,
        "value": round(value_gbs, 2),
        "unit": "GB/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": total_ms / args.steps,
        "us_per_call": per_call_s * 1e6,
        "hbm_frac_of_peak": kernel_gbs / peak,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u8 keys, f32 LUT/accumulate",
        "data": "synthetic (bench_cli generator: W=random_uniform(m,n,0x5EED), x=random_normal(n,b,0x5EED+1+j))",
        "config": {"workload": f"{args.config} m={m} n={n} q={beta} mu={mu} b={b}" + (
            f" per rank (layer {world * m}x{n}, y all-gathered with NCCL)" if world > 1 else ""),
                   "m": m, "n": n, "beta": beta, "mu": mu, "batch": b,
                   "step": "one BiQGEMM call (own weights copy, own x, own LUT build, y written)",
                   "l2": f"inputs larger than L2: {copies} rotating weight copies = "
                         f"{copies * tiled0.numel() / 1e6:.0f} MB > 2x126 MB",
                   "timing": f"CUDA graph of {n_launch} grouped launches ({G} independent calls each, "
                             f"{'stream form' if stream_form else 'single-call kernels'}), CUDA events",
                   "parallelism": f"rows x{world}"},
        "roofline": {"bound": "hbm", "achieved": round(kernel_gbs, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(kernel_gbs / peak, 4), "traffic": ncu_traffic(args.config),
                     "peak_kind": peak_kind, "algorithmic_bytes_per_launch": kb * min(G, args.steps),
                     "kernel": "biqgemm_stream_kernel + stream_finalize_kernel" if stream_form else "fast path"},
        "latency": {"us_per_call": round(lat_us, 3), "gbs": round(kb / (lat_us * 1e-6) / 1e9, 1),
                    "frac": round(kb / (lat_us * 1e-6) / 1e9 / peak, 4),
                    "form": "dependent-call regime: one single-call kernel per step, PDL-chained CUDA graph"},
        "e2e": {"value": round(e2e_gbs, 3), "unit": "GB/s", "h2d_bytes_per_step": int(x_h[0].nbytes),
                "d2h_bytes_per_step": int(m * b * 4), "us_per_call": e2e_s / args.steps * 1e6,
                "api": f"bqg_layers_forward_host, {GE} calls per synchronised API call "
                       "(H2D / grouped kernels / D2H pipelined inside the call in sub-groups ramping "
                       "sized by host I/O, C2: 64-128-256..128-64 calls; LayerGroup handle array built once)"},
        "gpu_launches": 2 * n_launch if stream_form else args.steps * 2,
        "clocks": clocks,
        "parity_rel_fro": rel,
    }
    if world > 1:
        line["allgather_ms_total"] = gather_ms
    if world == 1 and not args.no_comparators:
        line["comparators"] = comparators(bq, layer, w_shard, x_h, m, n, beta, b, mu, kb, dev)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.config, keys, alpha, x_h[0], m, n, beta, mu, b, args.cpu_seconds)
    if rank == 0:
        print(json.dumps(line), flush=True)
    for L in e2e_layers:
        L.close()
    if world > 1:
        dist.destroy_process_group()


def comparators(bq, layer, w, x_h, m, n, beta, b, mu, kb, dev, calls=200):
    """The paper's comparison points on this GPU (Table IV
    analog), device-timed per call with rotating copies > 2x L2: cuBLAS dense
    GEMV on the dequantized weights (fp32 and bf16), the reference's
    unpack-then-multiply method (gemm_unpack, GPU kernel) and the packed-word
    bandwidth probe.  Each is a reference point, not the product."""
    import torch

    out = {}
    s = torch.cuda.Stream(device=dev)

    def timeit(fns):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            for f in fns[:3]:
                f()
            s.synchronize()
            with torch.cuda.graph(g, stream=s):
                for f in fns:
                    f()
            g.replay()
            s.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            g.replay()
            e1.record(s)
        s.synchronize()
        return e0.elapsed_time(e1) * 1e3 / len(fns)

    keys, alpha, planes = layer.export(planes=True)
    wq = np.zeros((m, n), np.float32)  # dequantize(q) (quantize.hpp:61-74): sum_i alpha_i * B_i
    bits = np.unpackbits(planes.view(np.uint8).reshape(beta, m, -1), axis=2, bitorder="little")[:, :, :n]
    for i in range(beta):
        wq += alpha[i][:, None] * (2.0 * bits[i] - 1.0).astype(np.float32)
    x_d = [torch.from_numpy(x).to(dev) for x in x_h[:4]]
    for name, dt in (("cublas_fp32_gemv", torch.float32), ("cublas_bf16_gemv", torch.bfloat16)):
        w0 = torch.from_numpy(wq).to(dev).to(dt)
        nc = int(np.ceil(2 * L2_BYTES / (w0.numel() * w0.element_size()))) + 1
        ws_ = [w0] + [w0.clone() for _ in range(nc - 1)]
        xs_ = [xx.to(dt) for xx in x_d]
        ys_ = [torch.empty((m, b), device=dev, dtype=dt) for _ in range(nc)]
        us = timeit([(lambda j=j: torch.matmul(ws_[j % nc], xs_[j % len(xs_)], out=ys_[j % nc])) for j in range(calls)])
        wbytes = w0.numel() * w0.element_size()
        out[name] = {"us_per_call": round(us, 3), "weight_bytes": int(wbytes),
                     "weight_gbs": round(wbytes / (us * 1e-6) / 1e9, 1)}
        del ws_
    p0 = torch.from_numpy(planes.view(np.int32)).to(dev)
    nc = int(np.ceil(2 * L2_BYTES / (p0.numel() * 4))) + 1
    ps = [p0] + [p0.clone() for _ in range(nc - 1)]
    al = torch.from_numpy(alpha).to(dev)
    yy = [torch.empty((m, b), device=dev) for _ in range(nc)]
    if b <= 8 and n * b * 4 <= 200 * 1024:
        us = timeit([(lambda j=j: bq.gemm_unpack_device(ps[j % nc], al, x_d[j % len(x_d)], yy[j % nc], m, n, beta,
                                                        stream=torch.cuda.current_stream().cuda_stream))
                     for j in range(calls)])
        out["gemm_unpack_gpu"] = {"us_per_call": round(us, 3), "key_gbs": round(kb / (us * 1e-6) / 1e9, 1)}
    po = torch.empty(1184 * 512, device=dev)
    us = timeit([(lambda j=j: bq.bandwidth_probe_device(ps[j % nc], beta * m, n, x_d[0], po,
                                                        stream=torch.cuda.current_stream().cuda_stream))
                 for j in range(calls)])
    out["bandwidth_probe_gpu"] = {"us_per_call": round(us, 3), "key_gbs": round(kb / (us * 1e-6) / 1e9, 1),
                                  "what": "streaming read of the packed sign words (the key-stream roofline)"}
    return out


# ------------------------------------------------------------ CPU reference


def cpu_baseline(config, keys, alpha, x, m, n, beta, mu, b, seconds):
    """The reference's own biqgemm (oracle/_ref) on this host, single thread
    and all threads; bench_cli protocol (warmup, median of repeats)."""
    from oracle.oracle import Port, Reference, cpu_threads, reference

    kb = key_bytes(m, n, beta, mu)
    ref = reference()
    kind = "reference" if ref is not None else "port"
    if ref is None:
        return {"value": None, "unit": "GB/s", "cores": 0, "kind": "port",
                "sample": "oracle/_ref missing; no timing"}
    keys32 = np.ascontiguousarray(keys, np.uint32)
    nthreads = cpu_threads()
    best = None
    detail = {}
    for threads in sorted({1, nthreads}):
        secs, cs = ref.time_biqgemm(keys32, alpha, n, mu, x, threads=threads, warmup=1, repeats=1)
        reps = int(max(3, min(200, seconds / max(secs[0], 1e-6))))
        secs, cs = ref.time_biqgemm(keys32, alpha, n, mu, x, threads=threads, warmup=2, repeats=reps)
        med = float(np.median(secs))
        detail[str(threads)] = {"median_us": med * 1e6, "repeats": reps, "checksum": cs}
        if best is None or med < best[0]:
            best = (med, threads, reps)
    med, threads, reps = best
    return {"value": round(kb / med / 1e9, 4), "unit": "GB/s", "cores": threads, "kind": kind,
            "us_per_call": med * 1e6,
            "sample": f"{config}: median of {reps} reference biqgemm calls (plan_tiles budget max(32KiB, 2^mu*b*4B)), "
                      f"threads in {{1,{nthreads}}}, best shown",
            "per_threads": detail, "host_threads": nthreads}


def run_reference(args):
    rank, _, world = dist_env()
    if rank != 0:
        return
    import paper_2005_09904_b200.biqgemm as bq  # host RNG only (pinned == reference RNG)
    from oracle.oracle import reference

    ref = reference()
    m, n, beta, b, mu = CONFIGS[args.config]
    if ref is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libbqg_ref.so not built"}))
        return
    w = ref.random_uniform(m, n, SEED)
    x = ref.random_normal(n, b, SEED + 1)
    _, alpha, keys = ref.quantize_pack(w, beta, mu)
    kb = key_bytes(m, n, beta, mu)
    from oracle.oracle import cpu_threads

    nthreads = cpu_threads()
    # per step: one reference call; pick the faster thread count on a probe
    best_t, best_s = 1, None
    for threads in sorted({1, nthreads}):
        secs, _ = ref.time_biqgemm(keys, alpha, n, mu, x, threads=threads, warmup=1, repeats=3)
        s = float(np.median(secs))
        if best_s is None or s < best_s:
            best_t, best_s = threads, s
    steps = args.steps
    secs, cs = ref.time_biqgemm(keys, alpha, n, mu, x, threads=best_t, warmup=args.warmup, repeats=steps)
    total = float(np.sum(secs))
    val = kb * steps / total / 1e9
    line = {
        "metric": METRIC, "value": round(val, 5), "unit": "GB/s", "n_gpus": world, "steps": steps,
        "warmup": args.warmup, "ms_per_step": total / steps * 1e3, "us_per_call": total / steps * 1e6,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32 keys, f64 LUT/accumulate",
        "data": "synthetic (bench_cli generator)", "impl": "reference",
        "config": {"workload": f"{args.config} m={m} n={n} q={beta} mu={mu} b={b}", "m": m, "n": n, "beta": beta,
                   "mu": mu, "batch": b},
        "cpu_baseline": {"value": round(val, 5), "unit": "GB/s", "cores": best_t, "kind": "reference",
                         "sample": f"{steps} reference biqgemm calls ({args.config}), threads={best_t} of {nthreads}"},
        "e2e": {"value": round(val, 5), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "checksum": cs,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=50)
    ap.add_argument("--config", default="C2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-comparators", action="store_true", help="skip the cuBLAS / unpack / probe reference points")
    ap.add_argument("--batch", type=int, default=0, help="override the config's batch b (C4 sweep)")
    ap.add_argument("--group", type=int, default=128, help="independent calls per grouped launch")
    ap.add_argument("--e2e-group", type=int, default=512, help="calls per bqg_layers_forward_host call (e2e leg)")
    ap.add_argument("--profile", action="store_true", help="for ncu: warm-up + one timed replay only, no JSON line")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        args.steps = min(args.steps, 500)  # a reference step is ~30 ms of CPU: keep the run within minutes
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
