"""Per-CTA timeline of the fast kernel (BQG_DEBUG_FLAGS=2).
Slots: 0 start, 1 after griddepcontrol.wait, 2 first LUT built, 3 first key
stage landed, 4 query done, 5 smid, 6/7 last segment start / LUT built."""
import ctypes as C
import os
import sys
from pathlib import Path

os.environ["BQG_DEBUG_FLAGS"] = os.environ.get("BQG_DEBUG_FLAGS", "2")
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2005_09904_b200.biqgemm as bq  # noqa: E402
from bench import CONFIGS, SEED  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
NCOPIES = int(sys.argv[2]) if len(sys.argv) > 2 else 40
m, n, beta, b, mu = CONFIGS[cfg]
if len(sys.argv) > 3:
    b = int(sys.argv[3])
layer = bq.PackedLinear.from_weights(bq.random_uniform(m, n, SEED), beta, mu)
keys, alpha = layer.export()
tiled = bq.tile_keys(torch.from_numpy(keys).cuda(), n, mu)
copies = [tiled.clone() for _ in range(NCOPIES)]
al = torch.from_numpy(alpha).cuda()
x = torch.from_numpy(bq.random_normal(n, b, SEED + 1)).cuda()
y = torch.empty((m, b), device="cuda")
ws = bq.Workspace(int(bq.lib.bqg_biqgemm_workspace_bytes(m, n, b, beta, mu)))
CLUSTER = not (int(os.environ["BQG_DEBUG_FLAGS"]) & 128)
fn = bq.lib.bqg_debug_timeline_cluster if CLUSTER else bq.lib.bqg_debug_timeline
fn.argtypes = [C.c_void_p, C.c_int]
for i in range(30):
    bq.biqgemm_device(copies[i % NCOPIES], al, x, y, m, n, beta, mu, ws, pdl=os.environ.get('BQG_PDL', '1') == '1')
torch.cuda.synchronize()
W = 16 if CLUSTER else 8
t = np.zeros((8192, W), np.uint64)
fn(t.ctypes.data, 8192)
t = t[t[:, 0] > 0].astype(np.int64)
t0 = t[:, 0].min()
rel = {k: t[:, k] - t0 for k in range(5)}
print(f"{cfg} b={b}: CTAs {len(t)}  mode {'cluster' if CLUSTER else '2-kernel'}")
rows = [("start", rel[0]), ("pdl_wait", rel[1]), ("lut_built", rel[2]), ("keys_landed", rel[3]),
        ("query_done", rel[4]), ("d build", rel[2] - rel[1]), ("d query", rel[4] - rel[2])]
if CLUSTER:
    rows += [("cluster_bar", t[:, 6] - t0), ("first_out", t[:, 7] - t0), ("reduce_done", t[:, 5] - t0),
             ("d barrier", t[:, 6] - t[:, 4]), ("d reduce", t[:, 5] - t[:, 6])]
if CLUSTER and int(os.environ["BQG_DEBUG_FLAGS"]) & 1024:
    rows += [("lat x", t[:, 8]), ("lat keys", t[:, 9]), ("lat alpha", t[:, 10]), ("lat partial", t[:, 11])]
if CLUSTER:
    rows += [("bar_init", t[:, 14] - t0), ("syncthreads", t[:, 15] - t0), ("tma_issue0", t[:, 13] - t0),
             ("pre_pdlwait", t[:, 12] - t0)]
if not CLUSTER:
    two = t[:, 6] > 0
    print(f"CTAs with a second segment: {int(two.sum())}")
    if two.any():
        rows += [("seg2_start", t[two, 6] - t0), ("seg2_built", t[two, 7] - t0),
                 ("d seg2 build", t[two, 7] - t[two, 6]), ("d seg1 query", t[two, 6] - t[two, 2]),
                 ("d seg2 query", t[two, 4] - t[two, 7])]
for name, v in rows:
    print(f"{name:12s} min {v.min():7d} med {int(np.median(v)):7d} max {v.max():7d} ns")
