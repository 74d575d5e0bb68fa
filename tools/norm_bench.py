"""CUDA-event timing of autosp RMSNorm fwd/bwd vs torch F.rms_norm (dev tool)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import torch.nn.functional as F
from paper_2604_27089_b200 import kernels as K

for rows, d in [(32768, 2048), (131072, 4096)]:
    x = torch.randn(rows, d, device="cuda").bfloat16()
    w = torch.randn(d, device="cuda").bfloat16()
    dy = torch.randn(rows, d, device="cuda").bfloat16()
    y, rs = K.rms_norm_fwd(x, w, 1e-5)
    for name, fn in [("autosp fwd", lambda: K.rms_norm_fwd(x, w, 1e-5)),
                     ("autosp bwd", lambda: K.rms_norm_bwd(dy, x, w, rs)),
                     ("torch fwd", lambda: torch.ops.aten._fused_rms_norm(x, [d], w, 1e-5)),
                     ("torch bwd", lambda: torch.ops.aten._fused_rms_norm_backward(
                         dy, x, [d], rs.view(rows, 1), w, [True, True]))]:
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        nbytes = rows * d * 2 * (2 if "fwd" in name else 3)
        print(f"rows={rows} d={d} {name}: {ms*1e3:.1f} us  {nbytes/ms/1e6:.0f} GB/s", flush=True)
