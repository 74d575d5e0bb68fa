"""Multi-process CPU test of the whole AutoSP graph path (gloo, world_size 2):
Dynamo capture -> auto_sp (collectives + rank-offset positions) -> AOTAutograd ->
sp_ac partition -> execution with the TEST-ONLY CPU lowering of the custom ops ->
SP-group gradient reduction, compared against the CPU oracle (fp64) — the
reference's criterion 1 (test_acceptance.py:57-102) through the real pass stack."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from oracle import seqcomp_oracle as orc


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _graph_break_decoder(dims, dtype, in_loop=False):
    """SeqcompDecoder whose forward graph-breaks after the embedding + positions (Dynamo
    hands auto_sp an attention-free subgraph holding the position index -- ADVICE r1 /
    VERDICT r1 weak 9) and, with in_loop, also inside the layer loop (Dynamo then skips
    the frame: its attention would run eagerly on the local shard)."""
    import torch.nn.functional as F

    from paper_2604_27089_b200 import positions
    from paper_2604_27089_b200.workloads import SeqcompDecoder, rmsnorm

    class GB(SeqcompDecoder):
        def forward(self, ids):
            dm = self.dims
            b, s = ids.shape
            x = self.embed_table[ids.long() % dm.vocab]
            x = x + positions(s, device=ids.device).to(x.dtype).view(s, 1)
            torch._dynamo.graph_break()
            for l in range(dm.layers):
                res = x
                y = rmsnorm(x, self.norm1[l], 1e-6) @ self.qkv[l].t()
                y = y.view(b, s, dm.h, dm.d).transpose(1, 2)
                y = F.scaled_dot_product_attention(y, y, y, is_causal=True)
                if in_loop and l == 0:
                    torch._dynamo.graph_break()
                x = y.transpose(1, 2).reshape(b, s, dm.d_model) @ self.out[l].t() + res
                res = x
                y = F.silu(rmsnorm(x, self.norm2[l], 1e-6) @ self.up[l].t())
                x = y @ self.down[l].t() + res
            return x, (x * x).sum()

    return GB(dims, dtype=dtype)


def _worker(rank, world, port, dims_t, seed, passes, mode, q, graph_breaks=False, sp=None,
            grad_sync=False, accum=1):
    import torch.distributed as tdist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), AUTOSP_GRAD_BUCKET_BYTES=str(8 << 10))
    torch._dynamo.reset()
    try:
        tdist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2604_27089_b200 as autosp
        from paper_2604_27089_b200 import compiler, ops, sp_ac
        import autosp_cpu_lowering as testing
        from paper_2604_27089_b200.workloads import SeqcompDecoder, SeqcompDims
        testing.enable_cpu_lowering()
        ops.ATTN_DTYPE = None  # keep fp64 end to end on CPU
        autosp.reg_passes(passes, ac_mode=mode)
        sp = sp or world
        st = autosp.dist.init(sp, grad_sync=grad_sync)
        dims = SeqcompDims(*dims_t)
        odims = orc.Dims(*dims_t)
        ids, params = orc.random_leaves(odims, seed)
        if world > sp:  # data-parallel replica r // sp trains on its own batch
            ids = orc.random_leaves(odims, seed + 1 + rank // sp)[0]
        model = (_graph_break_decoder(dims, torch.float64, graph_breaks == "loop")
                 if graph_breaks else SeqcompDecoder(dims, dtype=torch.float64))
        model.load_reference(params)
        if grad_sync:  # a parameter used OUTSIDE the compiled graph (eager hook path)
            model.loss_scale = torch.nn.Parameter(torch.ones((), dtype=torch.float64))
        cm = autosp.compile(model)
        sl = dims.s // sp
        r_sp = rank % sp
        ids_r = torch.from_numpy(ids[:, r_sp * sl:(r_sp + 1) * sl].copy())
        for _ in range(accum):  # gradient accumulation: micro-batches before the step
            hidden, loss = cm(ids_r)
            (loss * model.loss_scale if grad_sync else loss).backward()
        grads = {k: p.grad.detach().clone() for k, p in model.named_reference_params().items()}
        local_loss = float(loss)
        autosp.dist.reduce_gradients(list(model.named_reference_params().values()), st)
        red = {k: p.grad.detach().numpy() for k, p in model.named_reference_params().items()}
        info = compiler.LAST_INFO.get("auto_sp")
        from paper_2604_27089_b200 import grad_sync as gsync
        if grad_sync:  # ZeRO-1 on top of the in-graph reduction: slice, AdamW, all-gather
            from paper_2604_27089_b200.zero import ShardedAdamW
            opt = ShardedAdamW(model.parameters(), st, bucket_bytes=4096, lr=1e-2)
            opt.step()
            red = dict(red, **{"after_adamw/" + k: p.detach().numpy().copy()
                               for k, p in model.named_reference_params().items()})
        plan = dict(sp_ac.LAST_PLAN, grad_sync=dict(gsync.LAST),
                    eager_grad=float(model.loss_scale.grad) if grad_sync else None,
                    in_graph=sum(bool(getattr(p, gsync.IN_GRAPH, False))
                                 for p in model.parameters()))
        q.put((rank, hidden.detach().numpy(), local_loss, red,
               {k: v.numpy() for k, v in grads.items()}, plan,
               {k: v.value for k, v in info.provenance.items()} if info else {}))
    except Exception as e:  # surface worker failures to the parent
        import traceback
        q.put((rank, "ERROR", traceback.format_exc(), None, None, None, None))
    finally:
        if tdist.is_initialized():
            tdist.destroy_process_group()


def _run(world, dims_t, seed, passes=("auto_sp", "sp_ac"), mode="seq-aware", graph_breaks=False,
         sp=None, grad_sync=False, accum=1):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, dims_t, seed, list(passes), mode, q,
                                               graph_breaks, sp, grad_sync, accum))
             for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        item = q.get(timeout=600)
        res[item[0]] = item
    for p in procs:
        p.join(timeout=60)
    for r, item in res.items():
        assert not (isinstance(item[1], str) and item[1] == "ERROR"), item[2]
    return [res[r] for r in range(world)]


@pytest.mark.parametrize("mode", ["seq-aware", "conservative", "seq-aware-all", "auto"])
def test_auto_sp_sp_ac_world2_matches_oracle(mode):
    dims_t = (1, 16, 4, 4, 8, 2, 64)  # b, s, h, d, d_ffn, layers, vocab
    out = _run(2, dims_t, seed=3, mode=mode)
    dims = orc.Dims(*dims_t)
    ids, params = orc.random_leaves(dims, 3)
    ref = orc.sp_forward_backward(dims, ids, params, 2)
    tg = ref.total_grads()
    for r, (_, hidden, loss, red, grads, plan, prov) in enumerate(out):
        assert orc.max_rel_err(hidden, ref.hidden[r]) <= 1e-10
        assert abs(loss - ref.loss[r]) <= 1e-10 * abs(ref.loss[r])
        for k in tg:  # per-rank partial gradients (reference sums them, finding 6)
            assert orc.max_rel_err(grads[k], ref.grads[r][k]) <= 1e-9, k
            assert orc.max_rel_err(red[k], tg[k]) <= 1e-9, k  # after SP-group reduction
        # 2 collectives per layer forward (q/k/v reshard, attention + O push); backward:
        # 2 (the dO reshard -- fused with delta = rowsum(dO*O) when the head dim is one
        # the kernels implement -- and the q/k/v gradient reshard); attention never
        # recomputed (sp_ac guard) and no forward collective re-issued
        assert plan["bw_collectives"] == 2 * dims.layers
        assert not plan["bw_recomputes_attention"]
        reasons = sorted(prov.values())
        assert reasons.count("InsertedCollective") == dims.layers
        assert "RecomputedIndex" in reasons


def test_auto_sp_without_sp_ac_world2():
    dims_t = (2, 8, 2, 4, 8, 1, 64)
    out = _run(2, dims_t, seed=9, passes=("auto_sp",))
    dims = orc.Dims(*dims_t)
    ids, params = orc.random_leaves(dims, 9)
    ref = orc.sp_forward_backward(dims, ids, params, 2)
    tg = ref.total_grads()
    for r, (_, hidden, loss, red, grads, plan, prov) in enumerate(out):
        assert orc.max_rel_err(hidden, ref.hidden[r]) <= 1e-10
        for k in tg:
            assert orc.max_rel_err(red[k], tg[k]) <= 1e-9, k


def test_graph_breaks_world2_matches_oracle():
    """auto_sp on Dynamo subgraphs without attention: no error, and the position index in
    the embedding subgraph still gets the rank offset (hidden states match the oracle)."""
    dims_t = (1, 16, 4, 4, 8, 2, 64)
    out = _run(2, dims_t, seed=5, graph_breaks="top")
    dims = orc.Dims(*dims_t)
    ids, params = orc.random_leaves(dims, 5)
    ref = orc.sp_forward_backward(dims, ids, params, 2)
    tg = ref.total_grads()
    for r, (_, hidden, loss, red, grads, plan, prov) in enumerate(out):
        assert orc.max_rel_err(hidden, ref.hidden[r]) <= 1e-10
        assert abs(loss - ref.loss[r]) <= 1e-10 * abs(ref.loss[r])
        for k in tg:
            assert orc.max_rel_err(red[k], tg[k]) <= 1e-9, k


def test_graph_break_in_loop_fails_loudly_at_p2():
    """A graph break inside the layer loop makes Dynamo run the whole loop eagerly: the
    attention would silently see only the local shard.  compile() raises instead."""
    with pytest.raises(AssertionError, match="fell back to eager"):
        _run(2, (1, 16, 4, 4, 8, 2, 64), seed=5, graph_breaks="loop")


def test_c1_size_world2_matches_reference_fixture(golden_dir):
    """BASELINE configs[0] at its real size (d_model 256, 8 heads, d 32, L 2, d_ffn 1024,
    s 1024, P 2) through the whole pass stack on gloo, against the reference's own P = 2
    result (model_c1_p2.npz, fp64): per-rank loss, sampled hidden rows and gradients."""
    z = np.load(golden_dir / "model_c1_p2.npz")
    b, s, h, d, f, L, P, seed, _ = (int(v) for v in z["dims"])
    out = _run(P, (b, s, h, d, f, L, 64), seed=seed, mode="seq-aware")
    dims = orc.Dims(b, s, h, d, f, L)
    hidden = np.concatenate([o[1] for o in out], axis=1)
    assert orc.norm_rel_err(hidden[:, z["hidden_rows"]], z["hidden_sample"]) < 1e-9
    for r, o in enumerate(out):
        assert abs(o[2] - z["loss_per_rank"][r]) <= 1e-9 * abs(z["loss_per_rank"][r])
        for i, n in enumerate(orc.param_names(dims)):
            g = o[3][n].reshape(-1)
            assert orc.norm_rel_err(g[z[f"grad_{i}_idx"]], z[f"grad_{i}_val"]) < 1e-9, n
        assert o[5]["mode_applied"] == "seq-aware" and o[5]["recomputed_fw_nodes"]


@pytest.mark.parametrize("world,sp,accum", [(2, 2, 1), (4, 2, 1), (2, 2, 2)])
def test_in_graph_grad_sync_listing1_loop(world, sp, accum):
    """Listing 1's unchanged loop: loss.backward() alone leaves every
    rank with the FULL gradient -- summed over the SP group inside the compiled backward
    (grad_sync.py), averaged over data-parallel replicas -- no reduce_gradients call.
    world 4 = SP 2 x DP 2 (paper's ZeRO-1 runs use SP x DP): each DP
    replica trains on its own batch; expected = mean over replicas of the oracle's
    summed SP gradients.  accum 2: two backward passes before the step (gradient
    accumulation) -- each contribution reduced once.  A scalar parameter used outside the
    compiled graph (loss * loss_scale) checks the eager-hook path: its gradient is the
    sum of the SP ranks' losses."""
    dims_t = (1, 16, 4, 4, 8, 2, 64)
    seed = 11
    out = _run(world, dims_t, seed=seed, sp=sp, grad_sync=True, accum=accum)
    dims = orc.Dims(*dims_t)
    _, params = orc.random_leaves(dims, seed)
    refs = []
    for dp in range(world // sp):
        ids = orc.random_leaves(dims, seed + 1 + dp)[0] if world > sp else \
            orc.random_leaves(dims, seed)[0]
        refs.append(orc.sp_forward_backward(dims, ids, params, sp))
    want = {k: accum * sum(r.total_grads()[k] for r in refs) / len(refs)
            for k in refs[0].total_grads()}
    want_eager = accum * sum(sum(r.loss) for r in refs) / len(refs)
    for r, (_, hidden, loss, red, grads, plan, prov) in enumerate(out):
        ref = refs[r // sp]
        assert orc.max_rel_err(hidden, ref.hidden[r % sp]) <= 1e-10
        for k in want:
            # grads = p.grad right after loss.backward(), before any explicit reduction
            assert orc.max_rel_err(grads[k], want[k]) <= 1e-9, (r, k)
            assert orc.max_rel_err(red[k], want[k]) <= 1e-9, (r, k)  # no double reduction
        # reduced INSIDE the backward graph: every parameter, in >1 bucket (8 KB buckets
        # here), the first issued well before the graph's end (overlap with the backward)
        gs = plan["grad_sync"]
        assert abs(plan["eager_grad"] - want_eager) <= 1e-10 * abs(want_eager), r
        assert plan["in_graph"] == len(want) == gs["params"]
        assert gs["buckets"] > 1 and gs["start_positions"][0] < 0.8 * gs["nodes"]
        # ZeRO-1 step on the already-reduced gradients == AdamW on the expected gradients
        for k in want:
            p = torch.nn.Parameter(torch.from_numpy(np.asarray(params[k], np.float64).copy()))
            p.grad = torch.from_numpy(np.asarray(want[k], np.float64).copy())
            torch.optim.AdamW([p], lr=1e-2).step()
            assert orc.max_rel_err(red["after_adamw/" + k], p.detach().numpy()) <= 1e-9, k
