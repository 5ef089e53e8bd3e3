"""e2e (bqg_layers_forward_host, 128 calls per API call) for one sub-group
schedule (BQG_E2E_SCHEDULE env, read by the library).  python tools/e2e_sched.py [steps]"""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2005_09904_b200.biqgemm as bq  # noqa: E402
from bench import CONFIGS, SEED, L2_BYTES  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 40
m, n, beta, b, mu = CONFIGS["C2"]
G = 128
layer = bq.PackedLinear.from_weights(bq.random_uniform(m, n, SEED), beta, mu)
keys, alpha = layer.export()
nl = int(np.ceil(4 * L2_BYTES / bq.tiled_key_bytes(m, n, beta, mu))) + 1
layers = [layer] + [bq.PackedLinear.from_keys(keys, alpha, n, mu) for _ in range(nl - 1)]
x_pin = torch.from_numpy(np.stack([bq.random_normal(n, b, SEED + 1 + i) for i in range(G)])).pin_memory()
y_pin = torch.empty((G, m, b), dtype=torch.float32).pin_memory()
groups = [bq.LayerGroup([layers[(s * G + i) % nl] for i in range(G)]) for s in range(8)]
for g in groups[:3]:
    bq.layers_forward_into(g, x_pin, y_pin)
best = []
for rep in range(5):
    t0 = time.perf_counter()
    for s in range(K):
        bq.layers_forward_into(groups[s % 8], x_pin, y_pin)
    best.append((time.perf_counter() - t0) / (K * G) * 1e6)
print(f"{os.environ.get('BQG_E2E_SCHEDULE', 'default'):24s} e2e us/call median {np.median(best):.3f} min {min(best):.3f}")
