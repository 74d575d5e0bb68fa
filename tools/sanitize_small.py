"""Small-shape driver for compute-sanitizer (racecheck / synccheck / memcheck) over the
hot kernels: K3 attention forward, K4 backward (d = 64 and 128, GQA, ragged s), and
the K1/K2 push kernel through a 4-virtual-rank loopback round trip (handshake, push,
wait, epoch flags).  Prints one line per part; run as
  compute-sanitizer --tool racecheck python tools/sanitize_small.py"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2604_27089_b200 import kernels as K

torch.manual_seed(0)
for (hq, hkv, s, d) in [(2, 1, 256, 64), (2, 2, 200, 128)]:
    q = torch.randn(1, hq, s, d, device="cuda").bfloat16()
    k = torch.randn(1, hkv, s, d, device="cuda").bfloat16()
    v = torch.randn(1, hkv, s, d, device="cuda").bfloat16()
    do = torch.randn(1, hq, s, d, device="cuda").bfloat16()
    o, lse = K.attn_fwd(q, k, v)
    dq, dk, dv = K.attn_bwd(q, k, v, o, do, lse)
    torch.cuda.synchronize()
    print(f"attention fwd+bwd hq={hq} hkv={hkv} s={s} d={d}: finite="
          f"{bool(torch.isfinite(dq.float()).all() and torch.isfinite(o.float()).all())}", flush=True)
shards = [torch.randn(1, 64, 8, 64, device="cuda").bfloat16() for _ in range(4)]
back = K.a2a_loopback("head_to_seq", K.a2a_loopback("seq_to_head", shards))
torch.cuda.synchronize()
print("a2a loopback round trip bit-exact:", all(torch.equal(a, b) for a, b in zip(back, shards)))
