"""ZeRO-1 over the SP group (zero.ShardedAdamW), gloo world size 2: reduce-scatter of the
per-rank partial gradients + AdamW on the owned shards + all-gather must equal plain
torch AdamW on the summed gradients (AdamW is elementwise), with chunking that splits
parameters across chunk and shard boundaries."""

import os
import socket

import numpy as np
import pytest
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


def _worker(rank, world, sp, port, q):
    import torch.distributed as tdist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2604_27089_b200 import dist, zero
        st = dist.init(sp)
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


@pytest.mark.parametrize("world,sp", [(2, 2), (4, 2)])
def test_sharded_adamw_equals_adamw_on_summed_grads(world, sp):
    """world 4 = SP 2 x DP 2 (the paper's SP x DP ZeRO-1 runs): the
    reduce-scatter over the SP group is followed by the mean over the DP group."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, sp, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, vals, sbytes = q.get(timeout=300)
        res[r] = (vals, sbytes)
    for p in procs:
        p.join(timeout=60)
    ref = [torch.nn.Parameter(t.clone()) for t in _init()]
    opt = torch.optim.AdamW(ref, lr=1e-2, weight_decay=0.1)
    dp = world // sp
    for step in range(3):
        gs = [_grads(r, step) for r in range(world)]
        for i, p in enumerate(ref):
            p.grad = sum(gs[r][i] for r in range(world)) / dp  # sum over SP, mean over DP
        opt.step()
    total = sum(int(np.prod(s)) for s in SHAPES)
    for r in range(world):
        for got, want in zip(res[r][0], ref):
            np.testing.assert_allclose(got, want.detach().numpy(), rtol=1e-12, atol=1e-12)
        # each rank holds ~1/SP of the shard values + 2 moments (fp64), not the full model
        assert res[r][1] <= 3 * 8 * (total // sp + 48)
