"""CUDA-event timing of one AdamW step over the Llama-3.2-1B parameter set (bf16):
optim.AdamW (multi-tensor kernel) vs torch.optim.AdamW(fused=True) (dev tool)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2604_27089_b200.optim import AdamW
from paper_2604_27089_b200.workloads import CONFIGS, LlamaDecoder

cfg = CONFIGS["llama3.2-1b"]
for name in ("torch", "autosp"):
    m = LlamaDecoder(cfg, dtype=torch.bfloat16, device="cuda")
    ps = list(m.parameters())
    for p in ps:
        p.grad = torch.randn_like(p)
    opt = torch.optim.AdamW(ps, lr=1e-4, fused=True) if name == "torch" else AdamW(ps, lr=1e-4)
    opt.step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        opt.step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    n = sum(p.numel() for p in ps)
    print(f"{name} AdamW: {ms:.2f} ms for {n / 1e9:.2f} B params, {14 * n / ms / 1e6:.0f} GB/s")
    del m, ps, opt
    torch.cuda.empty_cache()
