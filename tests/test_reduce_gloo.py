"""SP-group gradient reduction (dist.reduce_gradients, SURVEY §0 finding 6) over gloo,
world size 2, with buckets small enough that the packing, the oversized-gradient path and
mixed dtypes are all exercised."""

import os
import socket

import torch
import torch.multiprocessing as mp


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, port, q):
    import torch.distributed as tdist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE="2")
    tdist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        from paper_2604_27089_b200 import dist
        st = dist.init(2)
        shapes = [(3,), (64, 4), (5,), (2, 2), (300,), (7,)]
        dtypes = [torch.float32, torch.float32, torch.float64, torch.float64, torch.float32,
                  torch.float32]
        ps = []
        for i, (sh, dt) in enumerate(zip(shapes, dtypes)):
            p = torch.nn.Parameter(torch.zeros(sh, dtype=dt))
            p.grad = torch.full(sh, float(rank + 1) * (i + 1), dtype=dt)
            ps.append(p)
        dist.reduce_gradients(ps, st, bucket_bytes=256)
        q.put((rank, [p.grad.clone().numpy() for p in ps]))
    finally:
        tdist.destroy_process_group()


def test_bucketed_reduce_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    for r in range(2):
        for i, g in enumerate(res[r]):
            assert (g == 3.0 * (i + 1)).all(), (r, i, g.ravel()[:4])
