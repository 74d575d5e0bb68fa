"""CUDA-event timing of the SwiGLU kernels at the Llama-1B MLP shape (32K x 8192; dev tool)."""
import sys
sys.path.insert(0, '.')
import torch
from paper_2604_27089_b200 import kernels as K
gu = torch.randn(32768, 2 * 8192, device="cuda").bfloat16()
dout = torch.randn(32768, 8192, device="cuda").bfloat16()
for name, fn, nbytes in [("fwd", lambda: K.swiglu_fwd(gu), 3 * 32768 * 8192 * 2),
                         ("bwd", lambda: K.swiglu_bwd(gu, dout), 5 * 32768 * 8192 * 2)]:
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): fn()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"swiglu {name}: {ms*1e3:.1f} us {nbytes/ms/1e6:.0f} GB/s")
