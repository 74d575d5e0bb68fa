import sys, torch
sys.path.insert(0, "/root/repo")
from paper_2604_27089_b200 import kernels as K
d = torch.load(sys.argv[1])
q, k, v = d["q"], d["k"], d["v"]
print({n: (float(t.float().abs().max()), bool(torch.isfinite(t.float()).all())) for n, t in d.items() if torch.is_tensor(t)}, flush=True)
b, hq, s, hd = q.shape
hkv = k.shape[1]
qkv = torch.zeros(b, s, hq + 2 * hkv, hd, dtype=q.dtype, device="cuda")
qkv[:, :, hq + hkv:] = v.transpose(1, 2).cuda()
vv = qkv[:, :, hq + hkv:].transpose(1, 2)
qq = q.transpose(1, 2).contiguous().cuda().transpose(1, 2)
kk = k.transpose(1, 2).contiguous().cuda().transpose(1, 2)
for name, (a, bb, c) in {"model-data": (qq, kk, vv), "randn": (torch.randn_like(qq), torch.randn_like(kk), torch.randn_like(vv))}.items():
    o, lse = K.attn_fwd(a, bb, c, scale=d["scale"])
    torch.cuda.synchronize()
    print(name, "ok", float(o.float().abs().max()), flush=True)
