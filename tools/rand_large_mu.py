"""Randomised parity sweep of the mu > 8 fast path (re-keyed to mu = 8)
against the C oracle: random (m, n, beta, mu, b, x rows) incl. odd n, m not
a multiple of 32, x up to G*mu rows; single calls and a grouped host call.
python tools/rand_large_mu.py [cases]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

import paper_2005_09904_b200.biqgemm as bq  # noqa: E402
from oracle.oracle import port  # noqa: E402

P = port()
rng = np.random.default_rng(2024)
N = int(sys.argv[1]) if len(sys.argv) > 1 else 60
worst = 0.0
for case in range(N):
    m = int(rng.integers(1, 700))
    n = int(rng.integers(1, 3000))
    beta = int(rng.integers(1, 5))
    mu = int(rng.integers(9, 17))
    b = int(rng.choice([1, 1, 2, 3, 5, 8, 17, 33]))
    G = (n + mu - 1) // mu
    rows = int(rng.choice([n, max(1, n // 3), G * mu]))
    layer = bq.PackedLinear.from_weights(bq.random_uniform(m, n, 100 + case), beta, mu)
    keys, alpha = layer.export()
    x = bq.random_normal(rows, b, 200 + case)
    y = layer.forward(x)
    y_ref, _ = P.biqgemm(keys.astype(np.uint32), alpha, n, mu, x)
    rel = float(np.linalg.norm(y - y_ref) / max(np.linalg.norm(y_ref), 1e-30))
    mx = float(np.abs(y - y_ref).max() / max(np.abs(y_ref).max(), 1e-30))
    worst = max(worst, rel, mx)
    if rel > 1e-5 or mx > 1e-5:
        print(f"FAIL case {case}: m={m} n={n} beta={beta} mu={mu} b={b} rows={rows} rel={rel:.2e} max={mx:.2e}")
        sys.exit(1)
    if b == 1 and case % 4 == 0:
        xs = np.stack([bq.random_normal(rows, 1, 300 + case + i) for i in range(5)])
        yg = bq.layers_forward([layer] * 5, xs)
        for i in range(5):
            assert np.array_equal(yg[i], layer.forward(xs[i])), f"grouped != single, case {case}"
    layer.close()
print(f"rand_large_mu: {N} cases ok, worst relative error {worst:.2e}")
