"""CUDA-event timing of the chunked cross-entropy kernels at the Llama-3 vocabulary
(4096 tokens x 128256; dev tool)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2604_27089_b200 import _lib

lib = _lib.load()
n, V = 4096, 128256
logits = torch.randn(n, V, device="cuda").bfloat16()
labels = torch.randint(0, V, (n,), device="cuda")
lse = torch.empty(n, device="cuda")
loss = torch.empty(n, device="cuda")
st = torch.cuda.current_stream().cuda_stream
fn = lambda: lib.autosp_ce_fwd(logits.data_ptr(), labels.data_ptr(), lse.data_ptr(), loss.data_ptr(), n, V, V, st)
fn()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    fn()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
ref = torch.logsumexp(logits.float(), dim=1)
print(f"ce_fwd: {ms * 1e3:.1f} us {n * V * 2 / ms / 1e6:.0f} GB/s; max |lse - torch| {float((lse - ref).abs().max()):.2e}")
