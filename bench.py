#!/usr/bin/env python
"""BiQGEMM benchmark (driver contract: one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

Workload (N=1): BASELINE.json configs[1] = C2, the metric's own config:
GEMV m=n=4096, q(beta)=3 binary planes, mu=8, batch b=1, inputs generated
exactly like the reference's bench_cli (W = random_uniform(m,n,0x5EED),
x = random_normal(n,b,0x5EED+1)), quantized + packed ON THE GPU by the
product path.  A "step" is one BiQGEMM call (fused LUT build -> LUT query
-> alpha scale) on one layer's weights.

Timing (device): the K timed calls are captured in one CUDA graph with
programmatic dependent launch between consecutive calls (as consecutive
layers would run in a serving step) and replayed once between a
barrier+synchronize pair, timed with CUDA events on the replay stream.
Consecutive calls rotate over R distinct weight copies totalling > 2x the
126 MB L2, so every call streams its packed keys from HBM (inputs larger than
L2; no flush needed).  value = packed-key bytes of all ranks / max-over-ranks
time, in GB/s; us/call is reported beside it.

e2e: the same calls through the public C ABI with HOST buffers
(bqg_layer_forward_host: H2D of x from pinned memory, the kernel, D2H of y,
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

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for k, v in zip(names, s[3:7]):
                if "Active" in v and "Not" not in v:
                    reasons.add(k)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.samples)}


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


# ----------------------------------------------------------------------- ours


def run_ours(args):
    import torch
    import torch.distributed as dist

    rank, local_rank, world = dist_env()
    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    import paper_2005_09904_b200.biqgemm as bq

    m, n, beta, b, mu = CONFIGS[args.config]
    G = (n + mu - 1) // mu
    kb = key_bytes(m, n, beta, mu)  # per rank (weak scaling: each rank owns an m-row shard)
    dev = torch.device("cuda", local_rank)

    # ---- the layer: W generated like bench_cli, quantized + packed on the GPU
    m_total = m * world
    w = bq.random_uniform(m_total, n, SEED) if world > 1 else bq.random_uniform(m, n, SEED)
    w_shard = np.ascontiguousarray(w[rank * m:(rank + 1) * m])
    layer = bq.PackedLinear.from_weights(w_shard, beta, mu)
    keys, alpha = layer.export()
    x_h = bq.random_normal(n, b, SEED + 1)

    # ---- rotating weight copies > 2x L2
    tiled0 = torch.empty(bq.tiled_key_bytes(m, n, beta, mu), dtype=torch.uint8, device=dev)
    torch.cuda.synchronize()
    src = torch.from_numpy(keys).to(dev)
    tiled0.copy_(bq.tile_keys(src, n, mu))
    copies = max(2, int(np.ceil(2.0 * L2_BYTES / tiled0.numel())) + 1)
    tiled = [tiled0] + [tiled0.clone() for _ in range(copies - 1)]
    alphas = [torch.from_numpy(alpha).to(dev) for _ in range(copies)]
    x_d = torch.from_numpy(x_h).to(dev)
    ys = [torch.empty((m, b), device=dev) for _ in range(copies)]
    ws = bq.Workspace(int(bq.lib.bqg_biqgemm_workspace_bytes(m, n, b, beta, mu)), device=dev)
    stream = torch.cuda.Stream(device=dev)

    def call(i, s):
        j = i % copies
        bq.biqgemm_device(tiled[j], alphas[j], x_d, ys[j], m, n, beta, mu, ws, pdl=True, stream=s.cuda_stream)

    # ---- correctness gate before timing: y equals the exact path within tolerance
    with torch.cuda.stream(stream):
        call(0, stream)
    stream.synchronize()
    y_exact = layer.forward(x_h, exact=True)
    y0 = ys[0].cpu().numpy()
    rel = float(np.linalg.norm(y0.astype(np.float64) - y_exact) / np.linalg.norm(y_exact.astype(np.float64)))
    assert rel <= 1e-5, f"parity gate failed: rel {rel}"

    # ---- graphs: warmup (W calls) and timed (K calls)
    def capture(count, offset):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(stream):
            with torch.cuda.graph(g, stream=stream):
                for i in range(count):
                    call(offset + i, stream)
        return g

    g_warm = capture(max(args.warmup, 1), 0)
    g_timed = capture(args.steps, args.warmup)
    torch.cuda.synchronize()

    with ClockSampler(local_rank) as clk:
        # warm-up steps + enough untimed replays for steady clocks (>= 0.5 s)
        with torch.cuda.stream(stream):
            g_warm.replay()
            t0 = time.perf_counter()
            while time.perf_counter() - t0 < 0.5:
                g_timed.replay()
                stream.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            ev0.record(stream)
            g_timed.replay()
            ev1.record(stream)
        stream.synchronize()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ms = ev0.elapsed_time(ev1)
        clocks = clk.summary()

    # all-gather of y shards per step (N>1): timed separately as part of the step
    gather_ms = 0.0
    if world > 1:
        y_all = torch.empty((world * m, b), device=dev)
        for _ in range(3):
            dist.all_gather_into_tensor(y_all, ys[0])
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(args.steps):
            dist.all_gather_into_tensor(y_all, ys[i % copies])
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

    # ---- e2e through the public C ABI with host buffers (pinned)
    x_pin = torch.from_numpy(x_h).pin_memory()
    y_pin = torch.empty((m, b), dtype=torch.float32).pin_memory()
    e2e_layers = [layer] + [bq.PackedLinear.from_keys(keys, alpha, n, mu) for _ in range(copies - 1)]
    for i in range(max(args.warmup, 3)):
        e2e_layers[i % copies].forward_into(x_pin, y_pin)
    if world > 1:
        dist.barrier()
    e2e_steps = args.steps
    t0 = time.perf_counter()
    for i in range(e2e_steps):
        e2e_layers[i % copies].forward_into(x_pin, y_pin)
    e2e_s = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_s], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    assert np.allclose(y_pin.numpy(), y_exact, rtol=0, atol=1e-5 * np.abs(y_exact).max())
    e2e_gbs = world * kb * e2e_steps / e2e_s / 1e9

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
        "data": "synthetic (bench_cli generator: W=random_uniform(m,n,0x5EED), x=random_normal(n,b,0x5EED+1))",
        "config": {"workload": f"{args.config} m={m} n={n} q={beta} mu={mu} b={b}" + (
            f" per rank (layer {world * m}x{n}, y all-gathered with NCCL)" if world > 1 else ""),
                   "m": m, "n": n, "beta": beta, "mu": mu, "batch": b,
                   "l2": f"inputs larger than L2: {copies} rotating weight copies = "
                         f"{copies * tiled0.numel() / 1e6:.0f} MB > 2x126 MB",
                   "timing": "CUDA graph of K PDL-chained calls, CUDA events on the replay stream",
                   "parallelism": f"rows x{world}"},
        "roofline": {"bound": "hbm", "achieved": round(kernel_gbs, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(kernel_gbs / peak, 4), "traffic": ncu_traffic(args.config),
                     "peak_kind": peak_kind, "algorithmic_bytes_per_launch": kb},
        "e2e": {"value": round(e2e_gbs, 3), "unit": "GB/s", "h2d_bytes_per_step": int(x_h.nbytes),
                "d2h_bytes_per_step": int(m * b * 4), "us_per_call": e2e_s / e2e_steps * 1e6},
        "gpu_launches": args.steps,
        "clocks": clocks,
        "parity_rel_fro": rel,
    }
    if world > 1:
        line["allgather_ms_total"] = gather_ms
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.config, keys, alpha, x_h, m, n, beta, mu, b, args.cpu_seconds)
    if rank == 0:
        print(json.dumps(line), flush=True)
    for L in e2e_layers:
        L.close()
    if world > 1:
        dist.destroy_process_group()


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
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        args.steps = min(args.steps, 500)  # a reference step is ~30 ms of CPU: keep the run within minutes
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
