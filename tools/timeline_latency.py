"""Per-CTA timeline of the single-call latency kernel in a PDL chain
(BQG_DEBUG_FLAGS=2).  python tools/timeline_latency.py [C2|C4] [copies]"""
import ctypes as C
import os
import sys
from pathlib import Path

os.environ["BQG_DEBUG_FLAGS"] = "2"
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2005_09904_b200.biqgemm as bq  # noqa: E402
from bench import CONFIGS, SEED  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
NC = int(sys.argv[2]) if len(sys.argv) > 2 else 40
m, n, beta, b, mu = CONFIGS[cfg]
layer = bq.PackedLinear.from_weights(bq.random_uniform(m, n, SEED), beta, mu)
keys, alpha = layer.export()
t0 = bq.tile_keys(torch.from_numpy(keys).cuda(), n, mu)
copies = [t0.clone() for _ in range(NC)]
al = torch.from_numpy(alpha).cuda()
x = torch.from_numpy(bq.random_normal(n, b, SEED + 1)).cuda()
y = torch.empty((m, b), device="cuda")
ws = bq.Workspace(int(bq.lib.bqg_biqgemm_workspace_bytes(m, n, b, beta, mu)))
fn = bq.lib.bqg_debug_timeline_latency
fn.argtypes = [C.c_void_p, C.c_int]
for i in range(30):
    bq.biqgemm_device(copies[i % NC], al, x, y, m, n, beta, mu, ws, pdl=True)
torch.cuda.synchronize()
t = np.zeros((1024, 16), np.uint64)
fn(t.ctypes.data, 1024)
t = t[t[:, 0] > 0].astype(np.int64)
t0v = t[:, 0].min()
names = ["start", "cluster_arrive", "pdl_wait", "lut_built", "gathered", "pushed", "y_stored", "syncthreads",
         "w0_x_loaded", "w0_dfs_done", "w0_keys_1st", "w0_gathered", "keys_issued", "keys_all_landed"]
print(f"{cfg}: {len(t)} CTAs (last call of a 30-call PDL chain)")
for i, nm in enumerate(names):
    v = t[:, i] - t0v
    v = v[t[:, i] > 0]
    print(f"{nm:13s} min {v.min():7d} med {int(np.median(v)):7d} max {v.max():7d} ns")
