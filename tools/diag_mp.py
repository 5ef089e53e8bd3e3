"""Two processes sharing one GPU: single-call forwards of C2-shaped layers vs the oracle."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def worker(rank, q):
    import torch
    torch.cuda.set_device(0)
    import paper_2005_09904_b200.biqgemm as bq
    from oracle.oracle import Port
    port = Port()
    m, n, beta = 4096, 4096, 3
    bad = 0
    tot = 0
    for rep in range(4):
        for i in range(6):
            w = bq.random_uniform(m, n, 100 + i + 10 * rep)
            x = bq.random_normal(n, 1, 200 + i)
            f = bq.PackedLinear.from_weights(w, beta, 8)
            y = f.forward(x, exact=os.environ.get('DIAG_EXACT') == '1')
            keys, alpha = f.export()
            yp, _ = port.biqgemm(keys.astype(np.uint32), alpha, n, 8, x)
            rel = float(np.linalg.norm(y - yp) / np.linalg.norm(yp))
            tot += 1
            if rel > 1e-5:
                bad += 1
            f.close()
    q.put((rank, bad, tot, os.environ.get("BQG_DEBUG_FLAGS", "")))


if __name__ == "__main__":
    nproc = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=worker, args=(r, q)) for r in range(nproc)]
    for p in ps:
        p.start()
    for _ in range(nproc):
        print(q.get(timeout=600))
    for p in ps:
        p.join()
