"""Two processes sharing one GPU: where does a wrong forward come from?"""
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
    exact = os.environ.get("DIAG_EXACT") == "1"
    notes = []
    for rep in range(4):
        for i in range(6):
            w = bq.random_uniform(m, n, 100 + i + 10 * rep)
            x = bq.random_normal(n, 1, 200 + i)
            f = bq.PackedLinear.from_weights(w, beta, 8)
            y1 = f.forward(x, exact=exact)
            k1, a1 = f.export()
            y2 = f.forward(x, exact=exact)
            k2, a2 = f.export()
            yp, _ = port.biqgemm(k1.astype(np.uint32), a1, n, 8, x)
            pl, al = port.quantize_greedy(w, beta)
            kp = np.stack([port.pack_keys(pl[j], n, 8) for j in range(beta)])
            r1 = float(np.linalg.norm(y1 - yp) / np.linalg.norm(yp))
            r2 = float(np.linalg.norm(y2 - yp) / np.linalg.norm(yp))
            if r1 > 1e-5 or r2 > 1e-5 or not np.array_equal(k1, k2) or not np.array_equal(k1.astype(np.uint32), kp) or not np.array_equal(a1, al):
                notes.append(dict(rep=rep, i=i, r1=r1, r2=r2, keys_stable=bool(np.array_equal(k1, k2)),
                                  keys_vs_port=bool(np.array_equal(k1.astype(np.uint32), kp)),
                                  alpha_vs_port=bool(np.array_equal(a1, al)), y1_zero=bool(np.all(y1 == 0)),
                                  y1_nan=int(np.isnan(y1).sum()), y1_y2=bool(np.array_equal(y1, y2))))
            f.close()
    q.put((rank, notes))


if __name__ == "__main__":
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=worker, args=(r, q)) for r in range(2)]
    for p in ps:
        p.start()
    for _ in range(2):
        rank, notes = q.get(timeout=900)
        print(rank, len(notes))
        for nt in notes[:6]:
            print("   ", nt)
    for p in ps:
        p.join()
