"""µs per dependent call of a C2-sized layer (4096x4096, beta = 3, b = 1) for
mu in 1..8 through the layer handle (PDL-chained forward_device calls in a
CUDA graph, rotating layer copies > 2x L2): mu != 8 layers run on their sign
bits re-keyed to mu = 8 unless BQG_REKEY_SMALL_MU=0.  Parity against the
exact path of the same layer.  usage: python tools/small_mu_speed.py [mu ...]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2005_09904_b200.biqgemm as bq  # noqa: E402

m = n = 4096
beta = 3
mus = [int(a) for a in sys.argv[1:]] or [2, 4, 6, 7, 8]
w = bq.random_uniform(m, n, 3)
x = torch.from_numpy(bq.random_normal(n, 1, 4)).cuda()
s = torch.cuda.Stream()
for mu in mus:
    base = bq.PackedLinear.from_weights(w, beta, mu)
    keys, alpha = base.export()
    layers = [base] + [bq.PackedLinear.from_keys(keys, alpha, n, mu) for _ in range(12)]
    y = torch.empty((m, 1), device="cuda")
    ye = torch.empty((m, 1), device="cuda")
    base.forward_device(x, y)
    base.forward_device(x, ye, exact=True)
    torch.cuda.synchronize()
    rel = float(torch.linalg.norm(y - ye) / torch.linalg.norm(ye))
    K = 200
    with torch.cuda.stream(s):
        for L in layers:
            L.forward_device(x, y, pdl=True, stream=s.cuda_stream)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for i in range(K):
                layers[i % len(layers)].forward_device(x, y, pdl=True, stream=s.cuda_stream)
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
    print(f"mu={mu}: {np.median(ts):.2f} us per dependent call, rel_fro(fast, exact) {rel:.2e}")
    for L in layers:
        L.close()
