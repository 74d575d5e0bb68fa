"""auto_sp's fusion patterns on the Llama block's Dynamo graph (CPU, meta tensors, no
kernel runs): at P > 1 `h @ wqkv.t() -> view -> qkv_rope -> transpose -> SDPA` becomes ONE
`ulysses_qkv_proj_block` (K0 pushes RoPE'd rows from the GEMM epilogue) when K0's tile
constraints hold, and falls back to `ulysses_qkv_block` (cuBLAS GEMM + RoPE-fused K1)
when they do not (reference rewrite: sp_pass.py:172-195)."""

import pytest
import torch


class _Stop(Exception):
    pass


def _rewrite(seq_local, layers=2, world=2):
    from paper_2604_27089_b200 import dist, ops
    from paper_2604_27089_b200.auto_sp import auto_sp
    from paper_2604_27089_b200.workloads import LlamaConfig, LlamaDecoder
    st = dist.SPState(world=world, rank=1, name=f"pat{seq_local}")
    dist.register_state(st)
    cfg = LlamaConfig("pat", 256, layers, 4, 2, 512, 1000)  # d = 64, N = 8 * 64 = 512
    model = LlamaDecoder(cfg, dtype=torch.bfloat16, device="meta")
    seen = {}

    def backend(gm, example_inputs):
        gm, info = auto_sp(gm, example_inputs, st)
        seen["targets"] = [n.target for n in gm.graph.nodes if n.op == "call_function"]
        seen["methods"] = [n.target for n in gm.graph.nodes if n.op == "call_method"]
        seen["info"] = info
        raise _Stop

    torch._dynamo.reset()
    with pytest.raises(Exception) as ei:
        torch.compile(model, backend=backend)(torch.zeros(1, seq_local, dtype=torch.long,
                                                           device="meta"))
    assert "_Stop" in repr(ei.value) or isinstance(ei.value, _Stop), ei.value
    torch._dynamo.reset()
    return seen, ops


def test_qkv_projection_fused_into_k0():
    seen, ops = _rewrite(128)
    t = seen["targets"]
    assert t.count(ops.ulysses_qkv_proj_block) == 2 and seen["info"].fused_qkv_proj == 2
    assert ops.ulysses_qkv_block not in t
    assert torch.ops.autosp.qkv_rope.default not in t
    assert torch.nn.functional.scaled_dot_product_attention not in t
    # the projection matmul and its weight transpose are gone (the MLP's remain)
    assert "t" in seen["methods"] and seen["methods"].count("t") == 2 * 3


def test_qkv_projection_falls_back_outside_k0_tiles():
    seen, ops = _rewrite(64)  # s/P = 64: not a multiple of K0's 128-token tiles
    t = seen["targets"]
    assert t.count(ops.ulysses_qkv_block) == 2 and seen["info"].fused_qkv_proj == 0
    assert ops.ulysses_qkv_proj_block not in t
