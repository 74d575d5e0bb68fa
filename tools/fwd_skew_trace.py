"""Per-warp timeline of K3's first softmax warpgroup (tile 0 of the first CTA): when each of
its four warps releases S_0(j) and arrives P_0(j), relative to s_full.  Needs a library
built with -DAUTOSP_FWD_TRACE_SKEW=1 (tools/build_variant.py skew -DAUTOSP_FWD_TRACE_SKEW=1;
AUTOSP_LIB=tools/emu/libautosp_skew.so python tools/fwd_skew_trace.py)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2604_27089_b200 import _lib, kernels as K

lib = _lib.load()
s, d = 32768, 64
q = torch.randn(1, 32, s, d, device="cuda").bfloat16()
k = torch.randn(1, 8, s, d, device="cuda").bfloat16()
v = torch.randn(1, 8, s, d, device="cuda").bfloat16()
buf = torch.zeros(16 * 64, dtype=torch.int64, device="cuda")
lib.autosp_debug_set_fwd_trace(buf.data_ptr())
K.attn_fwd(q, k, v)
torch.cuda.synchronize()
lib.autosp_debug_set_fwd_trace(None)
t = buf.view(16, 64).cpu()
rel = lambda ev, j: int(t[ev, j] - t[4, j])
print("j: s_free(w0..w3) | p_arrive(w0..w3)   [cycles after sm0 s_full(j)]")
for j in range(8, 40):
    print(j, [rel(6 + w, j) for w in range(4)], [rel(10 + w, j) for w in range(4)])
sk = [max(rel(6 + w, j) for w in range(4)) - min(rel(6 + w, j) for w in range(4)) for j in range(8, 40)]
slow = [max(range(4), key=lambda w: rel(6 + w, j)) for j in range(8, 40)]
print("S-release skew per tile:", sk)
print("slowest warp per tile:", slow)
