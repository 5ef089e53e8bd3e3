"""Where does the time between grouped launches go?  Times CUDA graphs of L
back-to-back grouped launches (G calls each, rotating weight copies > 2x L2)
for L = 1, 2, 4, 16, and reports us/call; the slope over L is the steady
per-launch cost, the intercept the fill/drain.
python tools/launch_gap.py [C2|C4] [G]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2005_09904_b200.biqgemm as bq  # noqa: E402
from bench import CONFIGS, SEED, L2_BYTES  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
G = int(sys.argv[2]) if len(sys.argv) > 2 else 128
m, n, beta, b, mu = CONFIGS[cfg]
layer = bq.PackedLinear.from_weights(bq.random_uniform(m, n, SEED), beta, mu)
keys, alpha = layer.export()
t0 = bq.tile_keys(torch.from_numpy(keys).cuda(), n, mu)
copies = int(np.ceil(2.0 * L2_BYTES / t0.numel())) + 1
# one allocation for all copies: one texture window
big = torch.empty((copies, t0.numel()), dtype=torch.uint8, device="cuda")
for i in range(copies):
    big[i].copy_(t0)
al = torch.from_numpy(alpha).cuda()
xs = [torch.from_numpy(bq.random_normal(n, b, SEED + 1 + i)).cuda() for i in range(8)]
ys = [torch.empty((m, b), device="cuda") for _ in range(G)]
ws = bq.grouped_workspace(m, n, b, beta, mu, G)
s = torch.cuda.Stream()
k = 0


def launch_calls():
    global k
    ent = []
    for i in range(G):
        ent.append((big[k % copies], al, xs[k % 8], ys[i]))
        k += 1
    return bq.make_calls(ent)


for L in (1, 2, 4, 16):
    calls = [launch_calls() for _ in range(L)]
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        bq.biqgemm_grouped_device(calls[0], n, m, n, b, beta, mu, ws, pdl=True, stream=s.cuda_stream)
        s.synchronize()
        with torch.cuda.graph(g, stream=s):
            for c in calls:
                bq.biqgemm_grouped_device(c, n, m, n, b, beta, mu, ws, pdl=True, stream=s.cuda_stream)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            g.replay()
            e1.record(s)
        s.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"{cfg} G={G} launches={L:3d}: {best * 1e3:9.1f} us total  {best * 1e3 / (L * G):7.3f} us/call")
