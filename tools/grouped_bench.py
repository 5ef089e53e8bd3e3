"""Throughput of the grouped (stream) form vs the single-call PDL chain.
python tools/grouped_bench.py [C2|C4] [group] [m n beta]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2005_09904_b200.biqgemm as bq  # noqa: E402
from bench import CONFIGS, SEED, L2_BYTES, key_bytes  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
group = int(sys.argv[2]) if len(sys.argv) > 2 else 128
m, n, beta, b, mu = CONFIGS[cfg]
if len(sys.argv) > 5:  # shape override: python tools/grouped_bench.py C2 G m n beta
    m, n, beta = int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
kb = key_bytes(m, n, beta, mu)
layer = bq.PackedLinear.from_weights(bq.random_uniform(m, n, SEED), beta, mu)
keys, alpha = layer.export()
t0 = bq.tile_keys(torch.from_numpy(keys).cuda(), n, mu)
copies = int(np.ceil(2.0 * L2_BYTES / t0.numel())) + 1
tiled = [t0] + [t0.clone() for _ in range(copies - 1)]
al = [torch.from_numpy(alpha).cuda() for _ in range(copies)]
xs = [torch.from_numpy(bq.random_normal(n, b, SEED + 1 + i)).cuda() for i in range(copies)]
ys = [torch.empty((m, b), device="cuda") for _ in range(copies)]
y_ref = layer.forward(xs[0].cpu().numpy(), exact=True)
s = torch.cuda.Stream()
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731


def timeit(fn, reps=3):
    best = None
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = ev(), ev()
        with torch.cuda.stream(s):
            e0.record(s)
            fn()
            e1.record(s)
        s.synchronize()
        t = e0.elapsed_time(e1)
        best = t if best is None else min(best, t)
    return best


K = 2048
# single-call chain (graph)
ws1 = bq.Workspace(int(bq.lib.bqg_biqgemm_workspace_bytes(m, n, b, beta, mu)))
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    bq.biqgemm_device(tiled[0], al[0], xs[0], ys[0], m, n, beta, mu, ws1, pdl=True, stream=s.cuda_stream)
    s.synchronize()
    with torch.cuda.graph(g, stream=s):
        for i in range(K):
            j = i % copies
            bq.biqgemm_device(tiled[j], al[j], xs[j], ys[j], m, n, beta, mu, ws1, pdl=True, stream=s.cuda_stream)
g.replay()
ms = timeit(g.replay)
print(f"{cfg} single-call PDL chain : {ms * 1e3 / K:7.3f} us/call  {kb * K / ms / 1e6:8.1f} GB/s")


def grouped_graph(gsize, ws):
    gg = torch.cuda.CUDAGraph()
    calls = []
    for st in range(0, K, gsize):
        calls.append(bq.make_calls([(tiled[i % copies], al[i % copies], xs[i % copies], ys[i % copies])
                                    for i in range(st, min(K, st + gsize))]))
    with torch.cuda.stream(s):
        bq.biqgemm_grouped_device(calls[0], n, m, n, b, beta, mu, ws, pdl=True, stream=s.cuda_stream)
        s.synchronize()
        with torch.cuda.graph(gg, stream=s):
            for c in calls:
                bq.biqgemm_grouped_device(c, n, m, n, b, beta, mu, ws, pdl=True, stream=s.cuda_stream)
    return gg


for gsize in sorted({1, 32, 128, group}):
    ws = bq.grouped_workspace(m, n, b, beta, mu, gsize)
    gg = grouped_graph(gsize, ws)
    gg.replay()
    torch.cuda.synchronize()
    y0 = ys[0].cpu().numpy()
    rel = np.linalg.norm(y0.astype(np.float64) - y_ref) / np.linalg.norm(y_ref.astype(np.float64))
    ms = timeit(gg.replay)
    print(f"{cfg} grouped (group {gsize:4d})  : {ms * 1e3 / K:7.3f} us/call  {kb * K / ms / 1e6:8.1f} GB/s  rel {rel:.2e}")
