"""Kernel-time breakdown of one bench training step (torch.profiler / CUPTI; development
tool — numbers taken under a profiler are never bench values)."""
import argparse
import sys
from collections import defaultdict
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_2604_27089_b200 as autosp
from paper_2604_27089_b200.workloads import CONFIGS, LlamaConfig, LlamaDecoder, lm_loss

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="llama3.2-1b")
ap.add_argument("--seq", type=int, default=32768)
ap.add_argument("--layers", type=int, default=None)
ap.add_argument("--no-sp-ac", action="store_true")
ap.add_argument("--unfused", action="store_true")
a = ap.parse_args()
cfg = CONFIGS[a.model]
if a.layers:
    cfg = LlamaConfig(cfg.name, cfg.d_model, a.layers, cfg.hq, cfg.hkv, cfg.d_ffn, cfg.vocab)
autosp.reg_passes(["auto_sp"] if a.no_sp_ac else ["auto_sp", "sp_ac"])
autosp.dist.init(1)
torch.manual_seed(0)
m = LlamaDecoder(cfg, dtype=torch.bfloat16, device="cuda", fused=not a.unfused)
opt = torch.optim.AdamW(m.parameters(), lr=1e-4, fused=True)
cm = autosp.compile(m)
ids = torch.randint(0, cfg.vocab, (1, a.seq + 1), device="cuda")


def step():
    loss = lm_loss(cm(ids[:, :-1]), m.lm_head, ids[:, 1:])
    loss.backward()
    opt.step()
    opt.zero_grad(set_to_none=True)


for _ in range(3):
    step()
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    step()
    torch.cuda.synchronize()
tot = defaultdict(float)
cnt = defaultdict(int)
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        name = e.name.split("(")[0][:110]
        tot[name] += e.device_time_total / 1e3 if hasattr(e, "device_time_total") else e.cuda_time_total / 1e3
        cnt[name] += 1
T = sum(tot.values())
print(f"total kernel time {T:.1f} ms")
for n, v in sorted(tot.items(), key=lambda x: -x[1])[:40]:
    print(f"{v:9.2f} ms {100 * v / T:5.1f}% x{cnt[n]:4d}  {n}")
from paper_2604_27089_b200 import sp_ac
pl = sp_ac.LAST_PLAN
print("sp_ac:", {k: (v if not isinstance(v, list) else len(v)) for k, v in pl.items()})
print("bw ops:", pl.get("bw_recomputed_ops"))
