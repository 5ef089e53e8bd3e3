"""Small-shape driver for compute-sanitizer (memcheck / racecheck /
synccheck): the stream (grouped), latency (single call), cluster and
two-kernel forms, the exact path, the producers and the mu > 8 re-keying,
each once."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2005_09904_b200.biqgemm as bq  # noqa: E402

m, n, beta = 200, 700, 3
w = bq.random_uniform(m, n, 1)
layer = bq.PackedLinear.from_weights(w, beta, 8)
keys, alpha = layer.export()
for b in (1, 2, 5):
    x = bq.random_normal(n, b, 2)
    y = layer.forward(x)
    ye = layer.forward(x, exact=True)
    assert np.linalg.norm(y - ye) <= 1e-5 * np.linalg.norm(ye)
t = bq.tile_keys(torch.from_numpy(keys).cuda(), n, 8)
al = torch.from_numpy(alpha).cuda()
entries = [(t, al, torch.from_numpy(bq.random_normal(n, 1, 3 + i)).cuda(), torch.empty((m, 1), device="cuda"))
           for i in range(5)]
ws = bq.grouped_workspace(m, n, 1, beta, 8, 5)
bq.biqgemm_grouped_device(entries, n, m, n, 1, beta, 8, ws)
torch.cuda.synchronize()
# mu > 8: the re-keyed mu = 8 fast path (rekey + tile + the fast forms)
layer10 = bq.PackedLinear.from_weights(w, 2, 10)
for b in (1, 3):
    x = bq.random_normal(n, b, 9)
    y = layer10.forward(x)
    ye = layer10.forward(x, exact=True)
    assert np.linalg.norm(y - ye) <= 1e-5 * np.linalg.norm(ye)
torch.cuda.synchronize()
print("sanitize driver ok")
