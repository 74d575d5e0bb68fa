"""Quick CUDA-event timing of the attention kernels (development tool, not the bench)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2604_27089_b200 import kernels as K

def run(b, hq, hkv, s, d, iters=10):
    q = torch.randn(b, hq, s, d, device="cuda").bfloat16()
    k = torch.randn(b, hkv, s, d, device="cuda").bfloat16()
    v = torch.randn(b, hkv, s, d, device="cuda").bfloat16()
    do = torch.randn(b, hq, s, d, device="cuda").bfloat16()
    o, lse = K.attn_fwd(q, k, v)
    K.attn_bwd(q, k, v, o, do, lse)
    torch.cuda.synchronize()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record()
    for _ in range(iters):
        K.attn_fwd(q, k, v, out=o)
    e1.record()
    for _ in range(iters):
        K.attn_bwd(q, k, v, o, do, lse)
    e2.record()
    torch.cuda.synchronize()
    tf = e0.elapsed_time(e1) / iters
    tb = e1.elapsed_time(e2) / iters
    flops = 4.0 * b * hq * d * s * (s + 1) / 2  # causal fwd
    print(f"b={b} hq={hq} hkv={hkv} s={s} d={d}: fwd {tf:.3f} ms {flops/tf/1e9:.1f} TF/s | "
          f"bwd {tb:.3f} ms {2.5*flops/tb/1e9:.1f} TF/s", flush=True)

if __name__ == "__main__":
    for cfg in [(1, 32, 8, 32768, 64), (1, 4, 1, 32768, 64), (1, 32, 8, 8192, 128),
                (1, 4, 1, 131072, 128), (1, 8, 8, 16384, 128)]:
        run(*cfg)
