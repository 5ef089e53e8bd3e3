"""µs per call of K PDL-chained single calls in a CUDA graph (rotating weight
copies > 2x L2), no parity gate: for A/B runs with profiling switches
(BQG_DEBUG_FLAGS) that change what is computed.
usage: python tools/chain_time.py CFG [b] [K]"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2005_09904_b200.biqgemm as bq  # noqa: E402
from bench import CONFIGS, SEED  # noqa: E402

cfg = sys.argv[1]
m, n, beta, b, mu = CONFIGS[cfg]
if len(sys.argv) > 2 and int(sys.argv[2]) > 0:
    b = int(sys.argv[2])
K = int(sys.argv[3]) if len(sys.argv) > 3 else 50
G = (n + mu - 1) // mu
rng = np.random.default_rng(SEED)
keys = torch.from_numpy(rng.integers(0, 256, size=(beta, m, G), dtype=np.uint8)).cuda()
tiled = bq.tile_keys(keys, n, mu)
copies = max(2, int(np.ceil(2.5 * 126e6 / tiled.numel())))
tl = [tiled.clone() for _ in range(copies)]
al = torch.from_numpy(rng.uniform(0.01, 0.1, size=(beta, m)).astype(np.float32)).cuda()
x = torch.from_numpy(bq.random_normal(n, b, SEED + 1)).cuda()
y = torch.empty((m, b), device="cuda")
ws = bq.Workspace(int(bq.lib.bqg_biqgemm_workspace_bytes(m, n, b, beta, mu)))
s = torch.cuda.Stream()


def run(first, cnt):
    for i in range(first, first + cnt):
        bq.biqgemm_device(tl[i % copies], al, x, y, m, n, beta, mu, ws, pdl=True, stream=s.cuda_stream)


with torch.cuda.stream(s):
    run(0, 3)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        run(3, K)
    for _ in range(3):
        g.replay()
s.synchronize()
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s)
        g.replay()
        e1.record(s)
    s.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3 / K)
print(f"{cfg} b={b} flags={os.environ.get('BQG_DEBUG_FLAGS', '0')}: {np.median(ts):.2f} us/call (min {min(ts):.2f})")
