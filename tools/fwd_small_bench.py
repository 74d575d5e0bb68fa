import sys; sys.path.insert(0, '/root/repo')
import torch
from paper_2604_27089_b200 import kernels as K
for (hq, hkv, s, d) in [(32, 8, 32768, 64), (4, 1, 32768, 64), (4, 1, 16384, 64), (4, 1, 131072, 128)]:
    q = torch.randn(1, hq, s, d, device="cuda").bfloat16(); k = torch.randn(1, hkv, s, d, device="cuda").bfloat16(); v = torch.randn_like(k)
    o, lse = K.attn_fwd(q, k, v)
    for _ in range(3): K.attn_fwd(q, k, v, out=o)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 10
    e0.record()
    for _ in range(n): K.attn_fwd(q, k, v, out=o)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(f"fwd hq={hq} hkv={hkv} s={s} d={d}: {ms:.3f} ms {K.causal_attn_flops(1, hq, s, d)/ms/1e9:.1f} TF/s", flush=True)
