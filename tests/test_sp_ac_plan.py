"""sp_ac plan structure on a Llama-shaped graph (CPU, compile-time only: the partition
runs while tracing; execution is not needed).  The policy being pinned:
per layer the backward keeps the layer-input residual value, the attention output O
and its LSE — nothing O(s * d_ffn), no recomputed attention — so saved bytes grow
linearly in layers with a small per-layer constant (the reference's seq-aware guard set,
ac_pass.py:103-114, plus the AutoSP guards)."""

import pytest
import torch


def _plan(layers, s, mode="seq-aware"):
    torch._dynamo.reset()
    import paper_2604_27089_b200 as autosp
    from paper_2604_27089_b200 import sp_ac
    import autosp_cpu_lowering as testing
    from paper_2604_27089_b200.workloads import LlamaConfig, LlamaDecoder
    testing.enable_cpu_lowering()
    cfg = LlamaConfig("t", 256, layers, 4, 2, 512, vocab=128)
    autosp.reg_passes(["auto_sp", "sp_ac"], ac_mode=mode)
    autosp.dist.init(1)
    torch.manual_seed(0)
    m = LlamaDecoder(cfg, dtype=torch.float32, device="cpu", fused=False)
    cm = autosp.compile(m)
    out = cm(torch.randint(0, 128, (1, s)))
    out.sum().backward()
    return cfg, dict(sp_ac.LAST_PLAN)


@pytest.mark.parametrize("layers", [2, 8])
def test_seq_aware_keeps_one_residual_per_layer(layers):
    s = 256
    cfg, plan = _plan(layers, s)
    det = plan["saved_detail"]
    resid = [d for d in det if d[2] == (1, s, cfg.d_model)]
    attn_o = [d for d in det if d[2] == (1, cfg.hq, s, cfg.head_dim) and d[1] == "getitem"]
    lse = [d for d in det if d[2] == (1, cfg.hq, s)]
    ffn = [d for d in det if d[2][0] == 1 and (cfg.d_ffn in d[2][1:] or 2 * cfg.d_ffn in d[2][1:])]
    assert len(resid) == layers, resid
    assert len(attn_o) == layers and len(lse) == layers
    assert not ffn, ffn
    assert not plan["bw_recomputes_attention"]


def test_layer_boundary_detection_is_per_layer():
    """Deep graphs: the boundary search must stay in the forward graph (backward nodes
    reach everything), so every layer gets its checkpoint, not only the first few."""
    _, p2 = _plan(2, 128)
    _, p8 = _plan(8, 128)
    per_layer_2 = p2["saved_bytes"] / 2
    per_layer_8 = p8["saved_bytes"] / 8
    assert per_layer_8 < 1.5 * per_layer_2


@pytest.mark.parametrize("mode", ["seq-aware", "seq-aware-all", "conservative"])
def test_random_ops_are_never_recomputed(mode):
    """a recomputed dropout would draw a different mask in the backward than the
    forward used.  Random ops (Tag.nondeterministic_seeded) are guarded, so the backward
    graph contains none and the gradients equal eager autograd's under the same seed."""
    from functorch.compile import aot_function, make_boxed_func

    from paper_2604_27089_b200.sp_ac import AcMode, make_partition_fn
    bw_graphs = []

    def fw_c(gm, _):
        return make_boxed_func(gm.forward)

    def bw_c(gm, _):
        bw_graphs.append(gm)
        return make_boxed_func(gm.forward)

    def f(x, w1, w2):
        h = torch.nn.functional.dropout(x @ w1, p=0.5, training=True)
        return (torch.nn.functional.silu(h) @ w2).pow(2).sum()

    g = torch.Generator().manual_seed(0)
    x, w1, w2 = (torch.randn(*s, generator=g, dtype=torch.float64) for s in
                 ((64, 32), (32, 48), (48, 16)))
    cf = aot_function(f, fw_compiler=fw_c, bw_compiler=bw_c,
                      partition_fn=make_partition_fn(AcMode(mode)))
    leaves = [t.clone().requires_grad_(True) for t in (x, w1, w2)]
    torch.manual_seed(123)
    cf(*leaves).backward()
    ref = [t.clone().requires_grad_(True) for t in (x, w1, w2)]
    torch.manual_seed(123)
    f(*ref).backward()
    ops = {str(n.target) for n in bw_graphs[0].graph.nodes if n.op == "call_function"}
    rand = [o for o in ops if ("dropout" in o or "rand" in o or "bernoulli" in o)
            and "backward" not in o]
    assert not rand, ops
    for a, b in zip(leaves, ref):
        torch.testing.assert_close(a.grad, b.grad, rtol=1e-12, atol=1e-12)


def _seqcomp_plan(mode, dims_t=(1, 64, 4, 8, 32, 2, 64)):
    torch._dynamo.reset()
    import paper_2604_27089_b200 as autosp
    from paper_2604_27089_b200 import ops, sp_ac
    import autosp_cpu_lowering as testing
    from paper_2604_27089_b200.workloads import SeqcompDecoder, SeqcompDims
    testing.enable_cpu_lowering()
    ops.ATTN_DTYPE = None
    autosp.reg_passes(["auto_sp", "sp_ac"], ac_mode=mode)
    autosp.dist.init(1)
    torch.manual_seed(0)
    m = SeqcompDecoder(SeqcompDims(*dims_t), dtype=torch.float64)
    with torch.no_grad():
        for p in m.parameters():
            p.normal_(0.0, 0.1)
    _, loss = autosp.compile(m)(torch.randint(0, 64, (dims_t[0], dims_t[1])))
    loss.backward()
    return dict(sp_ac.LAST_PLAN)


MODES = ("conservative", "seq-aware", "seq-aware-all")


@pytest.mark.parametrize("model", ["seqcomp", "llama"])
def test_mode_cut_values_are_ordered(model):
    """Reference test_ac_pass.py:89-96: fewer guards can only lower the min cut --
    cut(seq-aware-all) <= cut(seq-aware) <= cut(conservative)."""
    if model == "seqcomp":
        cuts = {m: _seqcomp_plan(m)["cut_bytes"] for m in MODES}
    else:
        cuts = {m: _plan(2, 128, m)[1]["cut_bytes"] for m in MODES}
    assert cuts["seq-aware-all"] <= cuts["seq-aware"] <= cuts["conservative"], cuts


@pytest.mark.parametrize("mode", MODES)
def test_guards_never_recomputed(mode):
    """Reference test_ac_pass.py:98-105: no guarded forward node appears in the backward's
    recompute schedule; and the non-conservative modes do recompute something."""
    plan = _seqcomp_plan(mode)
    rec = set(plan["recomputed_fw_nodes"])
    assert not rec & set(plan["guarded"]), rec & set(plan["guarded"])
    assert plan["mode_applied"] == mode
    assert rec, "the plan recomputes nothing"
    assert not plan["bw_recomputes_attention"]
