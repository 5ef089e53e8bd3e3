"""Single-call time of the b >= 2 forms (biqgemm_fast_kernel + finalize),
device-resident, rotating weight copies > 2x L2, CUDA graph of PDL-chained
calls:  python tools/fast_sweep.py m n beta b [calls]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2005_09904_b200.biqgemm as bq  # noqa: E402
from bench import SEED, L2_BYTES, key_bytes  # noqa: E402

m, n, beta, b = (int(v) for v in sys.argv[1:5])
K = int(sys.argv[5]) if len(sys.argv) > 5 else 64
mu = 8
kb = key_bytes(m, n, beta, mu)
layer = bq.PackedLinear.from_weights(bq.random_uniform(m, n, SEED), beta, mu)
keys, alpha = layer.export()
t0 = bq.tile_keys(torch.from_numpy(keys).cuda(), n, mu)
copies = min(K, int(np.ceil(2.0 * L2_BYTES / t0.numel())) + 1)
tiled = [t0] + [t0.clone() for _ in range(copies - 1)]
al = torch.from_numpy(alpha).cuda()
x_h = bq.random_normal(n, b, SEED + 1)
x = torch.from_numpy(x_h).cuda()
y = torch.empty((m, b), device="cuda")
ws = bq.Workspace(int(bq.lib.bqg_biqgemm_workspace_bytes(m, n, b, beta, mu)))
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    bq.biqgemm_device(tiled[0], al, x, y, m, n, beta, mu, ws, pdl=True, stream=s.cuda_stream)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(K):
            bq.biqgemm_device(tiled[i % copies], al, x, y, m, n, beta, mu, ws, pdl=True, stream=s.cuda_stream)
g.replay()
torch.cuda.synchronize()
best = None
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s)
        g.replay()
        e1.record(s)
    s.synchronize()
    t = e0.elapsed_time(e1) / K
    best = t if best is None else min(best, t)
y_ref = layer.forward(x_h, exact=True)
rel = np.linalg.norm(y.cpu().numpy().astype(np.float64) - y_ref) / np.linalg.norm(y_ref)
lds_us = 4.0 * beta * m * ((n + 7) // 8) * b / (148 * 128 * 1.9e9) * 1e6
print(f"m={m} n={n} q={beta} b={b}: {best * 1e3:8.2f} us/call  (LDS roofline {lds_us:.1f} us = "
      f"{100 * lds_us / (best * 1e3):.0f}%)  rel {rel:.2e}")
