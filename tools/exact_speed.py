"""Speed of the exact path (fp64 tables in global memory) for mu = 8..16,
C2-sized layers (4096 x 4096, q = 3, b = 1), device-timed."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2005_09904_b200.biqgemm as bq  # noqa: E402

m = n = 4096
beta = 3
w = bq.random_uniform(m, n, 0x5EED)
x = torch.from_numpy(bq.random_normal(n, 1, 0x5EED + 1)).cuda()
for mu in (8, 10, 12, 14, 16):
    layer = bq.PackedLinear.from_weights(w, beta, mu)
    keys, alpha = layer.export()
    kd = torch.from_numpy(keys.view(np.int16) if mu > 8 else keys).cuda()
    ad = torch.from_numpy(alpha).cuda()
    y = torch.empty((m, 1), device="cuda")
    bq.biqgemm_exact_device(kd, ad, x, y, m, n, beta, mu)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        bq.biqgemm_exact_device(kd, ad, x, y, m, n, beta, mu)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 20
    kb = beta * m * ((n + mu - 1) // mu) * ((mu + 7) // 8)
    fast = ""
    if mu <= 8:
        fast = f"  (fast path: {layer.forward(x.cpu().numpy()) is not None})"
    print(f"mu={mu:2d} exact path {us:9.1f} us/call, keys {kb / 1e6:.2f} MB{fast}")
    layer.close()
