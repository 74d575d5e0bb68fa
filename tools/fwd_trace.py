"""Print the per-KV-tile pipeline timeline of the attention forward's heaviest CTA."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2604_27089_b200 import _lib, kernels as K

lib = _lib.load()
s = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
d = int(sys.argv[2]) if len(sys.argv) > 2 else 64
q = torch.randn(1, 32, s, d, device="cuda").bfloat16()
k = torch.randn(1, 8, s, d, device="cuda").bfloat16()
v = torch.randn(1, 8, s, d, device="cuda").bfloat16()
buf = torch.zeros(16 * 64, dtype=torch.int64, device="cuda")
lib.autosp_debug_set_fwd_trace(buf.data_ptr())
K.attn_fwd(q, k, v)
torch.cuda.synchronize()
lib.autosp_debug_set_fwd_trace(None)
t = buf.view(16, 64).cpu()
names = ["mma:p_full0", "mma:p_full1", "mma:o_done0", "mma:o_done1", "sm0:s_full", "sm1:s_full",
         "sm0:p_arrive", "sm1:p_arrive", "w0:parr", "w1:parr", "w2:parr", "w3:parr",
         "mma:s_free0", "mma:qk0_issued", "mma:v_full", "w0:s_free_arr"]
base = int(t[4, 0])
for j in range(10, 14):
    print(f"j={j}:")
    for i, n in enumerate(names):
        print(f"    {n:16s} {int(t[i, j]) - base:8d}")
print("per-tile cycles (sm0 s_full deltas):", [int(t[4, i + 1] - t[4, i]) for i in range(8, 40)])
print("sm0 softmax time per tile:", [int(t[6, i] - t[4, i]) for i in range(8, 24)])
