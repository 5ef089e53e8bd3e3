"""Parity of one fast-path form on assorted shapes (run in a subprocess with
BQG_DEBUG_FLAGS=8192 to force the cluster form or 128 for the two-kernel
form).  Exit code 0 = all shapes within the fp32 contract."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

import paper_2005_09904_b200.biqgemm as bq  # noqa: E402

shapes = [(4096, 4096, 3, 1), (1000, 4096, 2, 2), (2048, 2048, 3, 3), (513, 1100, 2, 4), (300, 3000, 1, 1),
          (64, 256, 3, 4), (4096, 3000, 2, 8), (777, 777, 3, 5)]
bad = 0
for m, n, beta, b in shapes:
    layer = bq.PackedLinear.from_weights(bq.random_uniform(m, n, m + n), beta, 8)
    x = bq.random_normal(n, b, m * 7 + b)
    y = layer.forward(x).astype(np.float64)
    ye = layer.forward(x, exact=True).astype(np.float64)
    rel = np.linalg.norm(y - ye) / np.linalg.norm(ye)
    mx = np.max(np.abs(y - ye)) / np.max(np.abs(ye))
    ok = rel <= 1e-5 and mx <= 1e-5 and np.array_equal(layer.forward(x), layer.forward(x))
    print(m, n, beta, b, f"rel={rel:.2e} max={mx:.2e}", "ok" if ok else "BAD")
    bad += 0 if ok else 1
    layer.close()
sys.exit(bad)
