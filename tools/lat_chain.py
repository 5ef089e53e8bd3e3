"""µs per call of K PDL-chained single calls (the latency form for these
shapes) in a CUDA graph, each call's x = the previous call's y (a true
dependent chain), rotating weight copies > 2x L2 (timing only: parity is the
-m gpu tests').  usage: python tools/lat_chain.py m n beta [K]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2005_09904_b200.biqgemm as bq  # noqa: E402

m, n, beta = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
K = int(sys.argv[4]) if len(sys.argv) > 4 else 200
assert m == n
mu = 8
G = (n + mu - 1) // mu
rng = np.random.default_rng(7)
keys = torch.from_numpy(rng.integers(0, 256, size=(beta, m, G), dtype=np.uint8)).cuda()
tiled = bq.tile_keys(keys, n, mu)
copies = max(2, int(np.ceil(2.5 * 126e6 / tiled.numel())))
tl = [tiled.clone() for _ in range(copies)]
# alpha ~ 1/(sqrt(n) * beta) keeps y of the chain O(1)
al = torch.from_numpy(rng.uniform(0.5, 1.5, size=(beta, m)).astype(np.float32) / (np.sqrt(n) * beta)).cuda()
xs = [torch.from_numpy(bq.random_normal(n, 1, 11)).cuda(), torch.empty((m, 1), device="cuda")]
ws = bq.Workspace(int(bq.lib.bqg_biqgemm_workspace_bytes(m, n, 1, beta, mu)))
form = int(bq.lib.bqg_biqgemm_form(m, n, 1, beta, mu))
s = torch.cuda.Stream()

def run(first, cnt):
    for i in range(first, first + cnt):
        bq.biqgemm_device(tl[i % copies], al, xs[i & 1], xs[(i + 1) & 1], m, n, beta, mu, ws, pdl=True,
                          stream=s.cuda_stream)


with torch.cuda.stream(s):
    run(0, 4)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        run(4, K)
    for _ in range(3):
        g.replay()
s.synchronize()
ts = []
for _ in range(7):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s)
        g.replay()
        e1.record(s)
    s.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3 / K)
print(f"m=n={m} beta={beta} form={form} K={K}: {np.median(ts):.3f} us/call (min {min(ts):.3f})")
