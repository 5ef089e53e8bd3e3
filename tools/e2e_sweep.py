"""End-to-end (host buffers) per-call time of bqg_layers_forward_host, the
bench.py e2e leg in isolation:  python tools/e2e_sweep.py [C2] [calls per API call]
(BQG_E2E_FIRST / BQG_E2E_SUB select the library's sub-group schedule)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2005_09904_b200.biqgemm as bq  # noqa: E402
from bench import CONFIGS, SEED, L2_BYTES, key_bytes  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
GE = int(sys.argv[2]) if len(sys.argv) > 2 else 512
steps = 2048
m, n, beta, b, mu = CONFIGS[cfg]
kb = key_bytes(m, n, beta, mu)
layer = bq.PackedLinear.from_weights(bq.random_uniform(m, n, SEED), beta, mu)
keys, alpha = layer.export()
copies = int(np.ceil(2.0 * L2_BYTES / kb)) + 1
layers = [layer] + [bq.PackedLinear.from_keys(keys, alpha, n, mu) for _ in range(copies - 1)]
x_pin = torch.from_numpy(np.stack([bq.random_normal(n, b, SEED + 1 + i) for i in range(GE)])).pin_memory()
y_pin = torch.empty((GE, m, b), dtype=torch.float32).pin_memory()
groups = [bq.LayerGroup([layers[(st + i) % copies] for i in range(min(GE, steps - st))]) for st in range(0, steps, GE)]
for grp in groups[:2]:
    bq.layers_forward_into(grp, x_pin[:len(grp)], y_pin[:len(grp)])
best = None
for _ in range(3):
    t0 = time.perf_counter()
    for grp in groups:
        bq.layers_forward_into(grp, x_pin[:len(grp)], y_pin[:len(grp)])
    t = time.perf_counter() - t0
    best = t if best is None else min(best, t)
y_ref = layer.forward(np.ascontiguousarray(x_pin[0].numpy()), exact=True)
assert np.allclose(y_pin[0].numpy(), y_ref, rtol=0, atol=1e-5 * np.abs(y_ref).max())
print(f"{cfg} e2e GE={GE}: {best / steps * 1e6:.3f} us/call  {kb * steps / best / 1e9:.1f} GB/s")

# where the time goes: device-side split of one API call (stats events) and
# the raw pinned copy rates
st = bq.KernelStats()
grp = groups[0]
t0 = time.perf_counter()
bq.layers_forward_into(grp, x_pin[:len(grp)], y_pin[:len(grp)], stats=st)
wall = time.perf_counter() - t0
print(f"  one API call of {len(grp)}: wall {wall * 1e6:.0f} us; kernels {st.query_seconds * 1e6:.0f} us; "
      f"copies outside the kernels {st.replace_seconds * 1e6:.0f} us")
for nb in (2 << 20, 8 << 20):
    h = torch.empty(nb // 4, dtype=torch.float32).pin_memory()
    d = torch.empty(nb // 4, dtype=torch.float32, device="cuda")
    for direction in ("h2d", "d2h"):
        for _ in range(2):
            (d.copy_(h, non_blocking=True) if direction == "h2d" else h.copy_(d, non_blocking=True))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(10):
            (d.copy_(h, non_blocking=True) if direction == "h2d" else h.copy_(d, non_blocking=True))
        torch.cuda.synchronize()
        t = (time.perf_counter() - t0) / 10
        print(f"  pinned {direction} {nb >> 20} MiB: {t * 1e6:.0f} us = {nb / t / 1e9:.1f} GB/s")
