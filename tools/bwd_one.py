"""A few attention-backward launches at the Llama-1B per-layer shape (s = 16K): the
target for `ncu --set full -k regex:attn_bwd_kernel` captures (dev tool)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2604_27089_b200 import kernels as K
b, hq, hkv, s, d = 1, 32, 8, 16384, 64
q = torch.randn(b, hq, s, d, device="cuda").bfloat16()
k = torch.randn(b, hkv, s, d, device="cuda").bfloat16()
v = torch.randn(b, hkv, s, d, device="cuda").bfloat16()
do = torch.randn(b, hq, s, d, device="cuda").bfloat16()
o, lse = K.attn_fwd(q, k, v)
for _ in range(2):
    K.attn_bwd(q, k, v, o, do, lse)
torch.cuda.synchronize()
