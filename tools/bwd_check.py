"""Quick numerics check of the attention backward against a torch fp32 reference at small
shapes (per-tensor relative errors); for kernel variants: AUTOSP_LIB=... python tools/bwd_check.py"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2604_27089_b200 import kernels as K


def ref(q, k, v, do, causal):
    q, k, v, do = (x.float().requires_grad_(x is not do) for x in (q, k, v, do))
    g = q.shape[1] // k.shape[1]
    kk, vv = k.repeat_interleave(g, 1), v.repeat_interleave(g, 1)
    s = q @ kk.transpose(-1, -2) / q.shape[-1] ** 0.5
    if causal:
        n = s.shape[-1]
        s = s.masked_fill(torch.ones(n, n, device=s.device).triu(1).bool(), float("-inf"))
    (s.softmax(-1) @ vv).backward(do)
    return q.grad, k.grad, v.grad


for (hq, hkv, s, d, causal) in [(2, 2, 128, 64, True), (2, 2, 256, 64, True), (2, 2, 256, 64, False),
                                (4, 2, 1024, 64, True), (2, 1, 1000, 64, True), (4, 2, 512, 32, True)]:
    torch.manual_seed(0)
    q = torch.randn(1, hq, s, d, device="cuda").bfloat16()
    k = torch.randn(1, hkv, s, d, device="cuda").bfloat16()
    v = torch.randn(1, hkv, s, d, device="cuda").bfloat16()
    do = torch.randn(1, hq, s, d, device="cuda").bfloat16()
    o, lse = K.attn_fwd(q, k, v, causal=causal)
    got = K.attn_bwd(q, k, v, o, do, lse, causal=causal)
    want = ref(q, k, v, do, causal)
    errs = [((a.float() - b).norm() / b.norm()).item() for a, b in zip(got, want)]
    print(f"hq={hq} hkv={hkv} s={s} d={d} causal={causal}: dq {errs[0]:.2e} dk {errs[1]:.2e} dv {errs[2]:.2e}")
