"""`biqgemm-bench`-compatible GPU harness.

Same flags, defaults, sweep order, timing protocol (warm-up, median of
repeats by wall time) and CSV schema as the reference's
/root/reference/proj/tools/bench_cli.cpp (flags 306-328, CSV 59-84,
run_scenario 97-176, run_verify 185-294), running the B200 library:

    python -m paper_2005_09904_b200.bench_cli --m 4096 --n 4096 --b 1 --beta 3 --mu 8 \\
        --method biqgemm,gemm_dense,gemm_unpack,bandwidth_probe --csv out.csv
    python -m paper_2005_09904_b200.bench_cli --verify --mu 2,4,8

Methods (host x in, host y out, like the reference's Matrix API):
  biqgemm          the fused BiQGEMM kernels (bqg_layer_forward_host)
  biqgemm_grouped  `--group` independent calls per API call (bqg_layers_forward_host);
                   wall_ms is per call
  gemm_dense       cuBLAS fp32 GEMM on dequantize(q) (baselines.hpp:14-36 analog)
  gemm_unpack      sum_i alpha_i * (B_i x) from the sign bits (baselines.hpp:40-52, GPU)
  bandwidth_probe  packed-word traffic only, values meaningless -> checksum NA
`threads` is recorded but has no effect on the GPU (KernelOptions::threads).
`budget-bytes` and `deterministic` are accepted for compatibility: the GPU
path is always deterministic and plans its own tiles.
"""
from __future__ import annotations

import argparse
import sys
import time

import numpy as np

from . import _capi
from . import biqgemm as bq

CSV_HEADER = ("m,n,b,beta,mu,threads,method,seed,repeats,warmup,"
              "wall_ms,build_ms,query_ms,replace_ms,"
              "lut_build_ops,lookups,accumulate_ops,fma_ops,checksum")
DEFAULT_SEED = 0x5EED
METHODS = ("biqgemm", "biqgemm_grouped", "gemm_dense", "gemm_unpack", "bandwidth_probe")


def _list(t):
    return lambda s: [t(v) for v in s.split(",") if v != ""]


def checksum(y) -> float:
    """bench_cli.cpp:36-40: sum of y in fp64, row-major order."""
    acc = 0.0
    for v in np.asarray(y, np.float32).reshape(-1):
        acc += float(v)
    return acc


def dequantize(planes, alpha, m, n):
    bits = np.unpackbits(planes.view(np.uint8).reshape(planes.shape[0], m, -1), axis=2, bitorder="little")[:, :, :n]
    w = np.zeros((m, n), np.float64)
    for i in range(planes.shape[0]):
        w += alpha[i].astype(np.float64)[:, None] * (2.0 * bits[i] - 1.0)
    return w.astype(np.float32)


def run_scenario(s, method, a):
    import torch

    m, n, b, beta, mu, threads = s
    w = bq.random_uniform(m, n, a.seed)
    x = bq.random_normal(n, b, a.seed + 1)
    layer = bq.PackedLinear.from_weights(w, beta, mu)
    keys, alpha, planes = layer.export(planes=True)
    G = bq.groups_of(n, mu)
    ops = dict(lut_build_ops=0, lookups=0, accumulate_ops=0, fma_ops=0)
    dev = torch.device("cuda")
    correct = True
    extra = {}
    if method == "biqgemm":
        y = np.empty((m, b), np.float32)

        def once(stats):
            layer.forward_into(x, y, stats=stats)
            return y
    elif method == "biqgemm_grouped":
        layers = [layer] + [bq.PackedLinear.from_keys(keys, alpha, n, mu) for _ in range(a.group - 1)]
        extra["layers"] = layers
        xs = np.ascontiguousarray(np.broadcast_to(x, (a.group, n, b)))
        ys = np.empty((a.group, m, b), np.float32)

        def once(stats):
            bq.layers_forward_into(layers, xs, ys, stats=stats)
            return ys[0]
    elif method == "gemm_dense":
        wd = torch.from_numpy(dequantize(planes, alpha, m, n)).to(dev)
        y = np.empty((m, b), np.float32)

        def once(stats):
            t0 = time.perf_counter()
            xd = torch.from_numpy(x).to(dev)
            t1 = time.perf_counter()
            yd = wd @ xd
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            y[...] = yd.cpu().numpy()
            t3 = time.perf_counter()
            stats.query_seconds += t2 - t1
            stats.replace_seconds += (t1 - t0) + (t3 - t2)
            stats.fma_ops += m * n * b
            return y
    elif method == "gemm_unpack":
        pd = torch.from_numpy(planes.view(np.int32)).to(dev)
        ad = torch.from_numpy(alpha).to(dev)
        y = np.empty((m, b), np.float32)
        if b > 8 or n * b * 4 > 200 * 1024:
            raise ValueError("gemm_unpack (GPU) needs b <= 8 and n*b*4 <= 200 KiB")

        def once(stats):
            t0 = time.perf_counter()
            xd = torch.from_numpy(x).to(dev)
            yd = torch.empty((m, b), device=dev)
            t1 = time.perf_counter()
            bq.gemm_unpack_device(pd, ad, xd, yd, m, n, beta)
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            y[...] = yd.cpu().numpy()
            t3 = time.perf_counter()
            stats.query_seconds += t2 - t1
            stats.replace_seconds += (t1 - t0) + (t3 - t2)
            stats.fma_ops += beta * m * n * b
            return y
    elif method == "bandwidth_probe":
        correct = False
        pd = torch.from_numpy(planes.view(np.int32)).to(dev)
        out = torch.empty(1184 * 512, device=dev)

        def once(stats):
            xd = torch.from_numpy(x).to(dev)
            bq.bandwidth_probe_device(pd, beta * m, n, xd, out)
            torch.cuda.synchronize()
            stats.fma_ops += beta * m * ((n + 31) // 32) * b
            return None
    else:
        raise ValueError(f"--method: unknown method {method}")

    for _ in range(a.warmup):
        once(bq.KernelStats())
    samples = []
    for _ in range(a.repeats):
        st = bq.KernelStats()
        t0 = time.perf_counter()
        yv = once(st)
        wall = time.perf_counter() - t0
        if method == "biqgemm_grouped":
            wall /= a.group
            for f in ("build_seconds", "query_seconds", "replace_seconds"):
                setattr(st, f, getattr(st, f) / a.group)
            for f in ("lut_build_ops", "lookups", "accumulate_ops", "fma_ops"):
                setattr(st, f, getattr(st, f) // a.group)
        samples.append((wall, st, checksum(yv) if (correct and yv is not None) else None))
    samples.sort(key=lambda t: t[0])
    wall, st, cs = samples[len(samples) // 2]
    for L in extra.get("layers", [layer])[1:]:
        L.close()
    layer.close()
    ops = dict(lut_build_ops=st.lut_build_ops, lookups=st.lookups, accumulate_ops=st.accumulate_ops,
               fma_ops=st.fma_ops)
    return dict(m=m, n=n, b=b, beta=beta, mu=mu, threads=threads, method=method, seed=a.seed, repeats=a.repeats,
                warmup=a.warmup, wall_ms=wall * 1e3, build_ms=st.build_seconds * 1e3, query_ms=st.query_seconds * 1e3,
                replace_ms=st.replace_seconds * 1e3, checksum=cs, **ops)


def write_record(out, r):
    out.write(f"{r['m']},{r['n']},{r['b']},{r['beta']},{r['mu']},{r['threads']},{r['method']},{r['seed']},"
              f"{r['repeats']},{r['warmup']},{r['wall_ms']:.4f},{r['build_ms']:.4f},{r['query_ms']:.4f},"
              f"{r['replace_ms']:.4f},{r['lut_build_ops']},{r['lookups']},{r['accumulate_ops']},{r['fma_ops']},"
              + ("NA" if r["checksum"] is None else f"{r['checksum']:.9e}") + "\n")


# ---------------------------------------------------------------- --verify


def run_verify(mus, seed, inject_pack_fault) -> int:
    """bench_cli.cpp:185-294 on the GPU library: codec bijection (with the
    mutation hook), DP vs naive tables, fast path vs dense reference and
    the counter laws on random shapes, footprint pins, model round trip.
    Returns the number of failures (the exit code)."""
    import torch

    for mu in mus:
        if mu < 1 or mu > 8:
            print(f"verify: mu={mu} out of range [1,8] for exhaustive checks", file=sys.stderr)
            return 2
    failures = 0

    def fail(msg):
        nonlocal failures
        print(f"FAIL: {msg}", file=sys.stderr)
        failures += 1

    rng = np.random.default_rng(seed)
    # codec bijection, exhaustive per mu: row k of a plane has the signs of key k
    for mu in mus:
        K = 1 << mu
        words = np.zeros((K, 1), np.uint32)
        for k in range(K):
            words[k, 0] = k  # bit t of row k = sign t (+1 where set), n = mu
        keys = bq.pack_keys(torch.from_numpy(words.view(np.int32)).cuda(), mu, mu).cpu().numpy().reshape(-1)
        keys = keys.astype(np.int64)
        if inject_pack_fault:
            keys = (keys + 1) % K
        if not np.array_equal(keys, np.arange(K)):
            fail(f"codec bijection violated at mu={mu}")
            if inject_pack_fault:
                break
    # DP vs naive (exact builders, lut.hpp:31-69)
    for mu in mus:
        xr = rng.standard_normal((mu, 1)).astype(np.float32)
        dp, _ = bq.build_lut_block(xr, 0, 1, mu, precision="f64")
        nv, _ = bq.build_lut_block(xr, 0, 1, mu, precision="f64", builder=_capi.LUT_NAIVE)
        if float((dp - nv).abs().max()) > 1e-12:
            fail(f"dp != naive at mu={mu}")
    # fast path vs dense reference + counter laws on 20 random shapes
    for _ in range(20):
        m, n, b = int(rng.integers(1, 200)), int(rng.integers(1, 300)), int(rng.integers(1, 6))
        beta, mu = int(rng.integers(1, 4)), int(rng.choice(mus))
        w = bq.random_uniform(m, n, int(rng.integers(0, 2**62)))
        x = bq.random_normal(n, b, int(rng.integers(0, 2**62)))
        layer = bq.PackedLinear.from_weights(w, beta, mu)
        keys, alpha, planes = layer.export(planes=True)
        st = bq.KernelStats()
        y = layer.forward(x, stats=st)
        ref = dequantize(planes, alpha, m, n).astype(np.float64) @ x.astype(np.float64)
        nrm = np.linalg.norm(ref)
        rel = np.linalg.norm(y - ref) / nrm if nrm > 0 else np.linalg.norm(y - ref)
        if rel > 1e-4:
            fail(f"biqgemm vs dense rel {rel:.3e} at m={m} n={n} b={b} beta={beta} mu={mu}")
        G = bq.groups_of(n, mu)
        if st.lookups != m * G * b * beta or st.lut_build_ops != ((1 << mu) + mu - 1) * G * b:
            fail("counter laws violated")
        layer.close()
    # footprint pins (model_io.cpp:182-194, Table II at 512 x 512)
    for bits, mb in ((32, 1.049), (8, 0.262), (6, 0.197), (4, 0.131), (3, 0.098), (2, 0.066)):
        f = bq.footprint(512, 512, bits)
        if abs(f.weight_mb() - mb) > 5e-4:
            fail(f"footprint {bits} bits: {f.weight_mb()} != {mb}")
    # model round trip (model_io.cpp:65-141)
    w = bq.random_uniform(40, 70, seed)
    layer = bq.PackedLinear.from_weights(w, 2, 4)
    keys, alpha = layer.export()
    data = bq.serialize_bqgm(keys, alpha, 40, 70, 2, 4)
    back = bq.PackedLinear.load(data)
    x = bq.random_normal(70, 2, seed + 1)
    if not np.array_equal(layer.forward(x), back.forward(x)):
        fail("model round trip changed the product")
    layer.close()
    back.close()
    print("verify: " + ("all checks passed" if failures == 0 else f"{failures} failure(s)"))
    return failures


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description="BiQGEMM benchmark harness (B200)")
    ap.add_argument("--m", type=_list(int), default=[1024], help="output sizes")
    ap.add_argument("--n", type=_list(int), default=[1024], help="input sizes")
    ap.add_argument("--b", type=_list(int), default=[32], help="batch sizes")
    ap.add_argument("--beta", type=_list(int), default=[1], help="quantization bits")
    ap.add_argument("--mu", type=_list(int), default=[8], help="LUT-unit sizes")
    ap.add_argument("--threads", type=_list(int), default=[1], help="worker counts (recorded; no effect on the GPU)")
    ap.add_argument("--method", type=_list(str), default=["biqgemm"], help="|".join(METHODS))
    ap.add_argument("--repeats", type=int, default=10, help="timed repeats (median reported)")
    ap.add_argument("--warmup", type=int, default=3, help="discarded warmup iterations")
    ap.add_argument("--seed", type=int, default=DEFAULT_SEED, help="RNG seed")
    ap.add_argument("--budget-bytes", type=int, default=32 * 1024, help="accepted for compatibility")
    ap.add_argument("--deterministic", action="store_true", help="accepted: the GPU path is always deterministic")
    ap.add_argument("--group", type=int, default=128, help="calls per API call for biqgemm_grouped")
    ap.add_argument("--csv", default="", help="write records to this file (default stdout)")
    ap.add_argument("--verify", action="store_true", help="run correctness self-checks and exit")
    ap.add_argument("--inject-pack-fault", action="store_true", help=argparse.SUPPRESS)
    a = ap.parse_args(argv)
    if a.repeats < 1:
        print("error: --repeats must be positive", file=sys.stderr)
        return 2
    if a.warmup < 0:
        print("error: --warmup must be non-negative", file=sys.stderr)
        return 2
    for mu in a.mu:  # bench_cli.cpp:332-337
        if mu < 1 or mu > 16:
            print(f"error: mu={mu} out of range [1,16]", file=sys.stderr)
            return 2
    if a.verify:
        return run_verify(a.mu, a.seed, a.inject_pack_fault)
    out = open(a.csv, "w") if a.csv else sys.stdout
    out.write(CSV_HEADER + "\n")
    try:
        for m in a.m:
            for n in a.n:
                for b in a.b:
                    for beta in a.beta:
                        for mu in a.mu:
                            for threads in a.threads:
                                for method in a.method:
                                    write_record(out, run_scenario((m, n, b, beta, mu, threads), method, a))
                                    out.flush()
    except (ValueError, _capi.BiqgemmError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 1
    finally:
        if a.csv:
            out.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
