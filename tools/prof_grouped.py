"""Driver for ncu: a few grouped launches of C2/C4-sized calls (distinct weights per call)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2005_09904_b200.biqgemm as bq  # noqa: E402
from bench import CONFIGS, SEED  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
count = int(sys.argv[2]) if len(sys.argv) > 2 else 16
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
m, n, beta, b, mu = CONFIGS[cfg]
layer = bq.PackedLinear.from_weights(bq.random_uniform(m, n, SEED), beta, mu)
keys, alpha = layer.export()
t0 = bq.tile_keys(torch.from_numpy(keys).cuda(), n, mu)
entries = [(t0.clone(), torch.from_numpy(alpha).cuda(), torch.from_numpy(bq.random_normal(n, b, SEED + 1 + i)).cuda(),
            torch.empty((m, b), device="cuda")) for i in range(count)]
ws = bq.grouped_workspace(m, n, b, beta, mu, count)
calls = bq.make_calls(entries)
for _ in range(reps):
    bq.biqgemm_grouped_device(calls, n, m, n, b, beta, mu, ws)
torch.cuda.synchronize()
print("done")
