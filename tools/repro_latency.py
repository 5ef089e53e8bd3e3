"""Minimal run of the single-call latency kernel (debugging aid)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2005_09904_b200.biqgemm as bq  # noqa: E402

m, n, beta = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (100, 300, 3)))
layer = bq.PackedLinear.from_weights(bq.random_uniform(m, n, 5), beta, 8)
keys, alpha = layer.export()
t = bq.tile_keys(torch.from_numpy(keys).cuda(), n, 8)
x = torch.from_numpy(bq.random_normal(n, 1, 6)).cuda()
y = torch.empty((m, 1), device="cuda")
ws = bq.Workspace(int(bq.lib.bqg_biqgemm_workspace_bytes(m, n, 1, beta, 8)))
bq.biqgemm_device(t, torch.from_numpy(alpha).cuda(), x, y, m, n, beta, 8, ws)
torch.cuda.synchronize()
ye = layer.forward(x.cpu().numpy(), exact=True)
print("rel", np.linalg.norm(y.cpu().numpy() - ye) / np.linalg.norm(ye))
