"""Print the per-step pipeline timeline of the attention backward's first CTA."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2604_27089_b200 import _lib, kernels as K

lib = _lib.load()
b, hq, hkv, s, d = 1, 32, 8, int(sys.argv[1]) if len(sys.argv) > 1 else 32768, int(sys.argv[2]) if len(sys.argv) > 2 else 64
q = torch.randn(b, hq, s, d, device="cuda").bfloat16()
k = torch.randn(b, hkv, s, d, device="cuda").bfloat16()
v = torch.randn(b, hkv, s, d, device="cuda").bfloat16()
do = torch.randn(b, hq, s, d, device="cuda").bfloat16()
o, lse = K.attn_fwd(q, k, v)
buf = torch.zeros(16 * 64, dtype=torch.int64, device="cuda")
lib.autosp_debug_set_bwd_trace(buf.data_ptr())
K.attn_bwd(q, k, v, o, do, lse)
torch.cuda.synchronize()
lib.autosp_debug_set_bwd_trace(None)
t = buf.view(16, 64).cpu()
names = ["mma:dq_empty", "mma:dP_issued", "mma:p_ready", "mma:ds_ready", "mma:dQ_issued",
         "sm:s_full", "sm:p_arrive", "sm:dp_full", "sm:ds_arrive", "dr:dq_full", "dr:dq_empty",
         "mma:q_next", "sm:loop_top", "mma:s_issued"]
base = int(t[1, 0])
for step in range(8, 16):
    row = "  ".join(f"{n}={int(t[i, step]) - base:8d}" for i, n in enumerate(names) if int(t[i, step]) > 0)
    print(f"t={step}: {row}")
print("per-step cycles (dP issue deltas):", [int(t[1, i + 1] - t[1, i]) for i in range(8, 40)])
print("per-step cycles (softmax loop-top deltas):", [int(t[12, i + 1] - t[12, i]) for i in range(8, 40)])
print("softmax wait for dP (dp_full - p_arrive):", [int(t[7, i] - t[6, i]) for i in range(8, 40)])
