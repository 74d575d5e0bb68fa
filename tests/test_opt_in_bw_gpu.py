"""Optimizer step inside the compiled backward on the Llama block (optim.AdamW, the bf16
multi-tensor kernel), one GPU: two training steps give BIT-IDENTICAL parameters to the
normal loop (backward, then optimizer.step()), every compiled parameter is updated inside
the graph (only the eager LM head by step()), and when the backward returns the compiled
parameters' gradients are already gone (the memory the normal loop holds until step())."""

import pytest
import torch

pytestmark = pytest.mark.gpu


def _run(in_backward: bool, mode: str):
    import paper_2604_27089_b200 as autosp
    from paper_2604_27089_b200 import opt_in_bw
    from paper_2604_27089_b200.optim import AdamW
    from paper_2604_27089_b200.workloads import LlamaConfig, LlamaDecoder, lm_loss
    torch._dynamo.reset()
    cfg = LlamaConfig("oib", 512, 2, 8, 4, 1024, 2048)
    autosp.reg_passes(["auto_sp", "sp_ac"], ac_mode=mode)
    autosp.dist.init(1)
    torch.manual_seed(0)
    model = LlamaDecoder(cfg, dtype=torch.bfloat16, device="cuda")
    opt = AdamW(model.parameters(), lr=1e-3)
    cm = autosp.compile(model, optimizer=opt if in_backward else None)
    g = torch.Generator().manual_seed(3)
    peaks, after_bwd = [], []
    for _ in range(2):
        ids = torch.randint(0, cfg.vocab, (1, 4097), generator=g).cuda()
        torch.cuda.synchronize()
        torch.cuda.reset_peak_memory_stats()
        loss = lm_loss(cm(ids[:, :-1]), model.lm_head, ids[:, 1:])
        loss.backward()
        torch.cuda.synchronize()
        peaks.append(torch.cuda.max_memory_allocated())
        after_bwd.append(torch.cuda.memory_allocated())
        n_grads = sum(p.grad is not None for p in model.parameters())
        opt.step()
        opt.zero_grad(set_to_none=True)
    torch.cuda.synchronize()
    params = [p.detach().clone() for p in model.parameters()]
    torch._dynamo.reset()
    grad_bytes = sum(p.numel() * p.element_size() for p in model.parameters()
                     if p is not model.lm_head)
    return params, (peaks, after_bwd, grad_bytes), n_grads, dict(opt_in_bw.LAST)


@pytest.mark.parametrize("mode", ["seq-aware", "auto"])
def test_optimizer_in_backward_bit_exact_and_frees_gradients(mode):
    ref, ref_peaks, ref_grads, _ = _run(False, mode)
    got, peaks, n_grads, info = _run(True, mode)
    for a, b in zip(got, ref):
        assert torch.equal(a, b)
    assert info["updated_in_graph"] == 2 * 6 + 2  # 6 weights per block + embedding + norm
    assert n_grads == 1 and ref_grads == 2 * 6 + 3  # only the eager LM head keeps a .grad
    (pk_ref, ab_ref, gbytes), (pk, ab, _) = ref_peaks, peaks
    print("after backward (normal, in-backward):", ab_ref[-1], ab[-1], "peak:", pk_ref[-1], pk[-1])
    if mode == "auto":  # save-all: nothing recomputed, the gradients are all that is freed
        assert ab[-1] <= ab_ref[-1] - 0.9 * gbytes, (ab, ab_ref, gbytes)
