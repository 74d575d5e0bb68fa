"""ZeRO-1 over the SP group (zero.ShardedAdamW), gloo world size 2: reduce-scatter of the
per-rank partial gradients + AdamW on the owned shards + all-gather must equal plain
torch AdamW on the summed gradients (AdamW is elementwise), with chunking that splits
parameters across chunk and shard boundaries."""

import os
import socket

import numpy as np
import torch
import torch.multiprocessing as mp


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


SHAPES = [(7, 5), (13,), (4, 4, 3), (33,), (2, 9)]


def _grads(rank, step):
    g = torch.Generator().manual_seed(100 * step + rank)
    return [torch.randn(sh, generator=g, dtype=torch.float64) for sh in SHAPES]


def _init():
    g = torch.Generator().manual_seed(0)
    return [torch.randn(sh, generator=g, dtype=torch.float64) for sh in SHAPES]


def _worker(rank, port, q):
    import torch.distributed as tdist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE="2")
    tdist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        from paper_2604_27089_b200 import dist, zero
        st = dist.init(2)
        ps = [torch.nn.Parameter(t.clone()) for t in _init()]
        opt = zero.ShardedAdamW(ps, st, bucket_bytes=8 * 24, lr=1e-2, weight_decay=0.1)
        assert len(opt.chunks) > 2  # chunk and shard boundaries cut through parameters
        for step in range(3):
            for p, g in zip(ps, _grads(rank, step)):
                p.grad = g.clone()
            opt.step()
            opt.zero_grad()
        q.put((rank, [p.detach().numpy().copy() for p in ps], opt.state_bytes()))
    finally:
        tdist.destroy_process_group()


def test_sharded_adamw_equals_adamw_on_summed_grads():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r, vals, sbytes = q.get(timeout=300)
        res[r] = (vals, sbytes)
    for p in procs:
        p.join(timeout=60)
    ref = [torch.nn.Parameter(t.clone()) for t in _init()]
    opt = torch.optim.AdamW(ref, lr=1e-2, weight_decay=0.1)
    for step in range(3):
        for p, g0, g1 in zip(ref, _grads(0, step), _grads(1, step)):
            p.grad = g0 + g1
        opt.step()
    total = sum(int(np.prod(s)) for s in SHAPES)
    for r in range(2):
        for got, want in zip(res[r][0], ref):
            np.testing.assert_allclose(got, want.detach().numpy(), rtol=1e-12, atol=1e-12)
        # each rank holds ~half the shard values + 2 moments (fp64), not the full model
        assert res[r][1] <= 3 * 8 * (total // 2 + 48)
