"""Generate the golden fixtures from the REFERENCE itself (oracle/_ref, the
unmodified reference headers compiled by oracle/Makefile).  Run here, where
/root/reference exists:

    python tests/golden/make_golden.py

Writes tests/golden/cases.npz (small randomized cases mirroring the
reference's acceptance generators), tests/golden/naive.npz (the same with
KernelOptions::builder = Naive) and tests/golden/configs.npz +
configs.json (the BASELINE configs' outputs/checksums on the bench_cli data,
seeds 0x5EED / 0x5EED+1, bench_cli.cpp:106-109).
"""
import json
import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))
from oracle.oracle import Reference  # noqa: E402

SEED = 0x5EED


def cases(ref):
    rng = np.random.Generator(np.random.PCG64(1234))
    out = {}
    idx = 0
    for mu in (1, 2, 3, 4, 5, 6, 7, 8, 9, 12, 16):
        for rep in range(3):
            m = int(rng.integers(1, 70))
            n = int(rng.integers(1, 90))
            b = int(rng.integers(1, 9))
            beta = int(rng.integers(1, 4))
            wseed, xseed = int(rng.integers(0, 2**63)), int(rng.integers(0, 2**63))
            w = ref.random_uniform(m, n, wseed)
            x = ref.random_normal(n, b, xseed)
            planes, alpha, keys = ref.quantize_pack(w, beta, mu)
            y, st = ref.biqgemm(keys, alpha, n, mu, x)
            yp, _ = ref.biqgemm(keys[:1], None, n, mu, x)
            G = keys.shape[2]
            lut_t, ops = ref.build_lut_block(x, 0, G, mu, key_major=False)
            lut_k, _ = ref.build_lut_block(x, 0, G, mu, key_major=True)
            p = f"c{idx}_"
            out[p + "dims"] = np.array([m, n, b, beta, mu, wseed, xseed], np.uint64)
            out[p + "planes"] = planes
            out[p + "alpha"] = alpha
            out[p + "keys"] = keys.astype(np.uint16)
            out[p + "y"] = y
            out[p + "yplane"] = yp
            if mu <= 9:  # keep the fixture small; larger tables are checked live
                out[p + "lut_t"] = lut_t
                out[p + "lut_k"] = lut_k
            out[p + "counters"] = np.array([st["lut_build_ops"], st["lookups"], st["accumulate_ops"]], np.uint64)
            idx += 1
    out["count"] = np.array([idx])
    np.savez_compressed(HERE / "cases.npz", **out)
    print("cases:", idx)


CONFIGS = {
    "C1": (1024, 1024, 1, 1),
    "C2": (4096, 4096, 3, 1),
    "C3": (4096, 4096, 2, 32),
    # BASELINE configs[3]: the full batch sweep 1..256
    **{f"C4b{b}": (16384, 4096, 3, b) for b in (1, 2, 4, 8, 16, 32, 64, 128, 256)},
    # BASELINE configs[4]: the multi-GPU config (row-sharded on the GPU side)
    "C5": (65536, 8192, 2, 8),
}
# Full y is stored when it is small; otherwise a strided row sample (<= ~16K
# floats) plus the sha256 of the reference's whole y (bytes of the f32 array)
# and its checksum.  The GPU exact path must reproduce y_sha bit-for-bit; the
# fast path is compared with that exact y (tests/test_gpu_parity.py).
SAMPLE_ELEMS = 16384


def configs(ref):
    import hashlib

    arrays, meta = {}, {}
    cache = {}
    for name, (m, n, beta, b) in CONFIGS.items():
        if (m, n, beta) not in cache:  # the C4 sweep shares W / keys
            cache.clear()
            w = ref.random_uniform(m, n, SEED)
            cache[(m, n, beta)] = (w,) + ref.quantize_pack(w, beta, 8)
        w, planes, alpha, keys = cache[(m, n, beta)]
        x = ref.random_normal(n, b, SEED + 1)
        # threads only split rows; the reference's result is bitwise
        # independent of them (acceptance criterion 7)
        y, st = ref.biqgemm(keys, alpha, n, 8, x, threads=os.cpu_count() or 1)
        stride = max(1, -(-(m * b) // SAMPLE_ELEMS))
        meta[name] = dict(m=m, n=n, beta=beta, b=b, mu=8, checksum=float(np.sum(y.astype(np.float64))),
                          y_sha=hashlib.sha256(np.ascontiguousarray(y).tobytes()).hexdigest(),
                          y_norm=float(np.linalg.norm(y.astype(np.float64))), sample_stride=stride,
                          lookups=st["lookups"], lut_build_ops=st["lut_build_ops"],
                          keys_sha=__import__("hashlib").sha256(keys.astype(np.uint8).tobytes()).hexdigest(),
                          alpha_sha=__import__("hashlib").sha256(alpha.tobytes()).hexdigest(),
                          w_sha=__import__("hashlib").sha256(w.tobytes()).hexdigest(),
                          x_sha=__import__("hashlib").sha256(x.tobytes()).hexdigest())
        if m * b <= 200_000:
            arrays[name + "_y"] = y
        else:
            arrays[name + "_ysample"] = np.ascontiguousarray(y[::stride])
        print(name, meta[name]["checksum"], flush=True)
    np.savez_compressed(HERE / "configs.npz", **arrays)
    (HERE / "configs.json").write_text(json.dumps(meta, indent=1))


def naive_cases(ref):
    """KernelOptions::builder = Naive (kernel.hpp:51,158; lut.hpp:31-43): the
    reference's y and counters with naive tables, next to its DP y."""
    rng = np.random.Generator(np.random.PCG64(4321))
    out = {}
    idx = 0
    for mu in (2, 3, 5, 8, 9, 11, 12):
        for rep in range(2):
            m = int(rng.integers(8, 200))
            n = int(rng.integers(16, 400))
            b = int(rng.integers(1, 5))
            beta = int(rng.integers(1, 4))
            wseed, xseed = int(rng.integers(0, 2**63)), int(rng.integers(0, 2**63))
            w = ref.random_uniform(m, n, wseed)
            x = ref.random_normal(n, b, xseed)
            _, alpha, keys = ref.quantize_pack(w, beta, mu)
            y_naive, st = ref.biqgemm(keys, alpha, n, mu, x, naive=True)
            y_dp, _ = ref.biqgemm(keys, alpha, n, mu, x)
            p = f"n{idx}_"
            out[p + "dims"] = np.array([m, n, b, beta, mu], np.uint64)
            out[p + "keys"] = keys.astype(np.uint16)
            out[p + "alpha"] = alpha
            out[p + "x"] = x
            out[p + "y_naive"] = y_naive
            out[p + "y_dp"] = y_dp
            out[p + "counters"] = np.array([st["lut_build_ops"], st["lookups"], st["accumulate_ops"]], np.uint64)
            idx += 1
    out["count"] = np.array([idx])
    np.savez_compressed(HERE / "naive.npz", **out)
    print("naive cases:", idx)


if __name__ == "__main__":
    r = Reference()
    if "--naive-only" in sys.argv:
        naive_cases(r)
        sys.exit(0)
    if "--configs-only" not in sys.argv:
        cases(r)
        naive_cases(r)
    configs(r)
