"""Wall time of the reference-style synchronous call (bqg_layer_forward_host,
pageable numpy x / y) for one layer, steady state."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

import paper_2005_09904_b200.biqgemm as bq  # noqa: E402

m, n, beta = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (4096, 4096, 3)))
layer = bq.PackedLinear.from_weights(bq.random_uniform(m, n, 0x5EED), beta, 8)
x = bq.random_normal(n, 1, 0x5EED + 1)
y = np.empty((m, 1), np.float32)
for _ in range(5):
    layer.forward_into(x, y)
t = []
for _ in range(200):
    t0 = time.perf_counter()
    layer.forward_into(x, y)
    t.append(time.perf_counter() - t0)
print(f"m={m} n={n} q={beta}: host forward median {np.median(t) * 1e6:.1f} us, min {np.min(t) * 1e6:.1f} us")
