"""Speed of the exact path (fp64 tables in global memory) and of the fast
path (mu > 8: the sign bits re-keyed to mu = 8) for mu = 8..16, C2-sized
layers (4096 x 4096, q = 3, b = 1), device-timed: the exact path 20 calls
back to back, the fast path 20 PDL-chained calls in a CUDA graph (one layer,
keys L2-resident: a per-call cost comparison, not a roofline)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2005_09904_b200.biqgemm as bq  # noqa: E402

m = n = 4096
beta = 3
w = bq.random_uniform(m, n, 0x5EED)
x_h = bq.random_normal(n, 1, 0x5EED + 1)
x = torch.from_numpy(x_h).cuda()


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


for mu in (8, 9, 10, 12, 14, 16):
    layer = bq.PackedLinear.from_weights(w, beta, mu)
    keys, alpha = layer.export()
    kd = torch.from_numpy(keys.view(np.int16) if mu > 8 else keys).cuda()
    ad = torch.from_numpy(alpha).cuda()
    y = torch.empty((m, 1), device="cuda")
    us_exact = timed(lambda: bq.biqgemm_exact_device(kd, ad, x, y, m, n, beta, mu))
    # the fast path as the layer runs it (x = n rows: the 8*ceil(n/8)-column
    # prefix of the re-keyed tiles), PDL-chained in a CUDA graph
    nf = 8 * ((n + 7) // 8) if mu > 8 else n
    ws = bq.Workspace(int(bq.lib.bqg_biqgemm_workspace_bytes(m, nf, 1, beta, 8 if mu > 8 else mu)))
    tk = torch.empty(0)
    s = torch.cuda.Stream()

    def fast():
        bq.lib.bqg_biqgemm_f32(layer.device_tiled_keys, layer.device_alpha, x.data_ptr(), n, y.data_ptr(), m, nf, 1,
                               beta, 8 if mu > 8 else mu, ws.ptr(), ws.nbytes, 1, s.cuda_stream)

    with torch.cuda.stream(s):
        fast()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(20):
                fast()
    s.synchronize()
    us_fast = timed(g.replay, reps=5) / 20
    layer.forward_device(x, y)
    torch.cuda.synchronize()
    y_fast = y.cpu().numpy().copy()
    y_exact = layer.forward(x_h, exact=True)
    rel = float(np.linalg.norm(y_fast - y_exact) / np.linalg.norm(y_exact))
    kb = beta * m * ((n + mu - 1) // mu) * ((mu + 7) // 8)
    print(f"mu={mu:2d} exact path {us_exact:9.1f} us/call (keys {kb / 1e6:.2f} MB)   fast path {us_fast:7.2f} us/call"
          f"   rel_fro(fast, exact) {rel:.2e}")
    layer.close()
