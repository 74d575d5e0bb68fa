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
         "sm0:p_arrive", "sm1:p_arrive", "tma:K_issue(j)", "tma:V_issue(j)", "mma0:k_full(j+1)ok", "mma0:k_full(j+1)wait",
         "mma0:s_free0", "mma0:qk0_issued", "mma0:v_full", "w0:s_free_arr"]
base = int(t[4, 0])
for j in range(10, 14):
    b = int(t[4, j])
    print(f"j={j}: (cycles after sm0:s_full of this tile)")
    for i in sorted(range(16), key=lambda i: int(t[i, j])):
        print(f"    {names[i]:18s} {int(t[i, j]) - b:8d}")
print("K(j+1) issue -> ready (tma:K_issue(j+1) -> mma0 k_full(j+1) passed):",
      [int(t[10, j] - t[8, j + 1]) for j in range(8, 40)])
print("per-tile cycles (sm0 s_full deltas):", [int(t[4, i + 1] - t[4, i]) for i in range(8, 40)])
print("sm0 softmax time per tile:", [int(t[6, i] - t[4, i]) for i in range(8, 24)])
