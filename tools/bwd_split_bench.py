"""K4 at the SP = 8 per-rank shapes (one kv head per rank: the small-grid case the GQA
split targets), with the split off (AUTOSP_BWD_HSPLIT=1) or automatic -- development tool.
  AUTOSP_BWD_HSPLIT=1 python tools/bwd_split_bench.py"""
import os
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2604_27089_b200 import kernels as K

for (hq, hkv, s, d) in [(32, 8, 32768, 64), (4, 1, 32768, 64), (4, 1, 131072, 128),
                        (4, 1, 16384, 64)]:
    q = torch.randn(1, hq, s, d, device="cuda").bfloat16()
    k = torch.randn(1, hkv, s, d, device="cuda").bfloat16()
    v = torch.randn_like(k)
    do = torch.randn_like(q)
    o, lse = K.attn_fwd(q, k, v)
    for _ in range(2):
        K.attn_bwd(q, k, v, o, do, lse)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 10 if s <= 32768 else 3
    e0.record()
    for _ in range(n):
        K.attn_bwd(q, k, v, o, do, lse)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(f"hsplit={os.environ.get('AUTOSP_BWD_HSPLIT', 'auto')} hq={hq} hkv={hkv} s={s} d={d}: "
          f"{ms:.3f} ms {2.5 * K.causal_attn_flops(1, hq, s, d) / ms / 1e9:.1f} TF/s", flush=True)
