"""optim.AdamW (multi-tensor bf16 kernel) against torch.optim.AdamW(fused=True) on the
same bf16 parameters and gradients: three steps with weight decay, ragged tensor sizes
(vector and scalar tails), more than one launch's worth of tensors.  Both compute in
fp32 and round to bf16, so they agree to bf16 rounding (stated: max |dp| <= 2 ulp of
the parameter scale)."""

import pytest
import torch

pytestmark = pytest.mark.gpu


def test_adamw_matches_torch():
    from paper_2604_27089_b200.optim import AdamW
    g = torch.Generator(device="cuda").manual_seed(0)
    shapes = [(1000,), (7,), (64, 33), (2048,), (129, 8)] * 15  # 75 tensors: two launches
    ref = [torch.randn(s, device="cuda", generator=g).bfloat16() for s in shapes]
    ours = [p.clone() for p in ref]
    ref = [torch.nn.Parameter(p) for p in ref]
    ours = [torch.nn.Parameter(p) for p in ours]
    kw = dict(lr=1e-2, betas=(0.9, 0.95), eps=1e-8, weight_decay=0.1)
    o_ref = torch.optim.AdamW(ref, fused=True, **kw)
    o_ours = AdamW(ours, **kw)
    for _ in range(3):
        for a, b in zip(ref, ours):
            gr = torch.randn(a.shape, device="cuda", generator=g).bfloat16()
            a.grad = gr.clone()
            b.grad = gr.clone()
        o_ref.step()
        o_ours.step()
    torch.cuda.synchronize()
    for a, b in zip(ref, ours):
        err = float((a.float() - b.float()).abs().max())
        scale = float(a.float().abs().max())
        assert err <= 2 * scale * 2 ** -8, (a.shape, err, scale)


def test_adamw_empty_tensors_and_distinct_steps():
    """zero-element tensors inside a 64-tensor batch must not shift the next
    batch (no tensor updated twice), and parameters with different step counts get their
    own bias corrections."""
    from paper_2604_27089_b200.optim import AdamW
    g = torch.Generator(device="cuda").manual_seed(1)
    shapes = [(0,), (100,)] * 40 + [(5,)] * 30  # 110 tensors, 40 of them empty
    ref = [torch.nn.Parameter(torch.randn(s, device="cuda", generator=g).bfloat16())
           for s in shapes]
    ours = [torch.nn.Parameter(p.detach().clone()) for p in ref]
    kw = dict(lr=1e-2, betas=(0.9, 0.95), eps=1e-8, weight_decay=0.1)
    o_ref, o_ours = torch.optim.AdamW(ref, fused=True, **kw), AdamW(ours, **kw)
    for it in range(3):
        # the first half of the tensors skip step 0, so their step counts lag by one
        for i, (a, b) in enumerate(zip(ref, ours)):
            if it == 0 and i < len(ref) // 2:
                a.grad = b.grad = None
                continue
            gr = torch.randn(a.shape, device="cuda", generator=g).bfloat16()
            a.grad, b.grad = gr.clone(), gr.clone()
        o_ref.step()
        o_ours.step()
    torch.cuda.synchronize()
    for a, b in zip(ref, ours):
        if a.numel() == 0:
            continue
        err = float((a.float() - b.float()).abs().max())
        scale = float(a.float().abs().max())
        assert err <= 2 * scale * 2 ** -8, (a.shape, err, scale)
