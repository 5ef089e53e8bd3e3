"""Diagnose the grouped row-sharded call on one GPU with 2 gloo ranks."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2005_09904_b200.biqgemm as bq
    from paper_2005_09904_b200.sharded import ShardedGroup, ShardedLinear, TorchCollectives

    m, n, beta, count = 4096, 4096, 3, 6
    coll = TorchCollectives()
    ws_ = [bq.random_uniform(m, n, 100 + i) for i in range(count)]
    shards = [ShardedLinear.from_weights(w, beta, 8, rank, world, coll) for w in ws_]
    grp = ShardedGroup(shards)
    x_h = np.stack([bq.random_normal(n, 1, 200 + i) for i in range(count)])
    fulls = [bq.PackedLinear.from_weights(w, beta, 8) for w in ws_]
    y_full = [f.forward(x_h[i]) for i, f in enumerate(fulls)]
    from oracle.oracle import Port
    port = Port()
    full_ok = []
    for i, f in enumerate(fulls):
        keys, alpha = f.export()
        yp, _ = port.biqgemm(keys.astype(np.uint32), alpha, n, 8, x_h[i])
        full_ok.append(float(np.linalg.norm(y_full[i] - yp) / np.linalg.norm(yp)))
    q.put((rank, [(-1, "full_vs_port", full_ok)]))
    out = []
    for rep in range(4):
        x = torch.from_numpy(x_h).cuda() if rank == 0 else torch.zeros((count, n, 1), device="cuda")
        yg = grp.gather_buffer(1)
        yg.fill_(float("nan"))
        y = grp.forward_device(x, yg).cpu().numpy()
        xs = x.cpu().numpy()
        bad = []
        for i in range(count):
            d = np.abs(y[i] - y_full[i])[:, 0]
            if not np.array_equal(y[i], y_full[i]):
                rows = np.nonzero(~(d == 0))[0]
                bad.append((i, int(rows.min()), int(rows.max()), len(rows), float(np.nanmax(d)), int(np.isnan(y[i]).sum())))
        out.append((rep, bool(np.array_equal(xs, x_h)), bad))
    q.put((rank, out))
    dist.destroy_process_group()


if __name__ == "__main__":
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=worker, args=(r, 2, 29611, q)) for r in range(2)]
    for p in ps:
        p.start()
    for _ in range(4):
        rank, out = q.get(timeout=300)
        for rep, xok, bad in out:
            print("rank", rank, "rep", rep, "x ok", xok, "bad", bad)
    for p in ps:
        p.join()
