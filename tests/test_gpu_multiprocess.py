"""Two processes sharing one GPU (time-sliced contexts): the FIRST forward of
a fresh layer must be right.  Regression test for a race between the
workspace's zero fill (once queued on the legacy default stream) and the
first kernels on the layer's non-blocking stream -- invisible in a single
process, a wrong or all-zero first y when another process delayed the fill."""
import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _worker(rank, exact, q):
    try:
        import torch

        torch.cuda.set_device(0)
        import paper_2005_09904_b200.biqgemm as bq
        from oracle.oracle import Port

        port = Port()
        m, n, beta = 4096, 4096, 3
        bad = []
        for i in range(8):
            w = bq.random_uniform(m, n, 100 + i + 31 * rank)
            x = bq.random_normal(n, 1, 200 + i)
            f = bq.PackedLinear.from_weights(w, beta, 8)
            y = f.forward(x, exact=exact)  # the first call on fresh buffers
            keys, alpha = f.export()
            yp, _ = port.biqgemm(keys.astype(np.uint32), alpha, n, 8, x)
            rel = float(np.linalg.norm(y - yp) / np.linalg.norm(yp))
            if rel > 1e-5:
                bad.append((i, rel))
            f.close()
        q.put((rank, bad))
    except Exception as e:  # report instead of leaving the parent waiting
        q.put((rank, [("error", repr(e))]))


@pytest.mark.parametrize("exact", [False, True])
def test_first_forward_with_a_second_process_on_the_gpu(cuda, exact):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, exact, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=600) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    for rank, bad in res:
        assert not bad, f"rank {rank}: {bad}"
