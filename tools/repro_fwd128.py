import sys, torch
sys.path.insert(0, "/root/repo")
from paper_2604_27089_b200 import kernels as K
for s in (4096, 32768):
    for d, hq, hkv in ((128, 32, 8), (64, 32, 8)):
        qkv = torch.randn(1, s, hq + 2 * hkv, d, device="cuda").bfloat16()
        q = qkv[:, :, :hq].contiguous().transpose(1, 2)          # like rope output
        k = qkv[:, :, hq:hq + hkv].contiguous().transpose(1, 2)
        v = qkv[:, :, hq + hkv:].transpose(1, 2)                  # strided slice of qkv
        try:
            o, lse = K.attn_fwd(q, k, v)
            torch.cuda.synchronize()
            print("ok", s, d, hq, hkv, flush=True)
        except Exception as e:
            print("FAIL", s, d, hq, hkv, e, flush=True)
            raise
