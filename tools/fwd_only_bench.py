"""CUDA-event timing of the attention forward alone (Llama-1B per-layer shape at 32K, or
argv: s d) -- for same-box A/B of kernel variants (AUTOSP_LIB=...)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2604_27089_b200 import kernels as K
s = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
d = int(sys.argv[2]) if len(sys.argv) > 2 else 64
hq, hkv = (32, 8) if d == 64 else (4, 1)
q = torch.randn(1, hq, s, d, device="cuda").bfloat16()
k = torch.randn(1, hkv, s, d, device="cuda").bfloat16()
v = torch.randn_like(k)
o, lse = K.attn_fwd(q, k, v)
for _ in range(3):
    K.attn_fwd(q, k, v, out=o)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 20 if s <= 32768 else 5
e0.record()
for _ in range(n):
    K.attn_fwd(q, k, v, out=o)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / n
print(f"fwd s={s} d={d}: {ms:.3f} ms {K.causal_attn_flops(1, hq, s, d) / ms / 1e9:.1f} TF/s")
