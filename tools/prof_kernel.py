"""Minimal driver for ncu: builds one config's layer and runs `--calls`
fast-path calls (no graph, no PDL) on rotating weight copies."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2005_09904_b200.biqgemm as bq  # noqa: E402
from bench import CONFIGS, SEED  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--calls", type=int, default=6)
ap.add_argument("--copies", type=int, default=4)
ap.add_argument("--b", type=int, default=0)
a = ap.parse_args()
m, n, beta, b, mu = CONFIGS[a.config]
if a.b:
    b = a.b
layer = bq.PackedLinear.from_weights(bq.random_uniform(m, n, SEED), beta, mu)
keys, alpha = layer.export()
tiled = bq.tile_keys(torch.from_numpy(keys).cuda(), n, mu)
tl = [tiled] + [tiled.clone() for _ in range(a.copies - 1)]
al = torch.from_numpy(alpha).cuda()
x = torch.from_numpy(bq.random_normal(n, b, SEED + 1)).cuda()
y = torch.empty((m, b), device="cuda")
ws = bq.Workspace(int(bq.lib.bqg_biqgemm_workspace_bytes(m, n, b, beta, mu)))
for i in range(a.calls):
    bq.biqgemm_device(tl[i % a.copies], al, x, y, m, n, beta, mu, ws)
torch.cuda.synchronize()
print("done", a.config, float(y.sum()))
