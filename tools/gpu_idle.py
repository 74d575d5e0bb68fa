"""GPU busy vs idle time inside one bench training step (torch.profiler / CUPTI kernel
timeline): sums kernel durations, finds the gaps between consecutive kernels on the GPU
and the largest of them (a CPU-bound / launch-bound stretch shows up as many gaps).
Development tool; profiler numbers are never bench values."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_2604_27089_b200 as autosp
from paper_2604_27089_b200.workloads import CONFIGS, LlamaDecoder, lm_loss

cfg = CONFIGS["llama3.2-1b"]
autosp.reg_passes(["auto_sp", "sp_ac"])
autosp.dist.init(1)
torch.manual_seed(0)
m = LlamaDecoder(cfg, dtype=torch.bfloat16, device="cuda")
opt = torch.optim.AdamW(m.parameters(), lr=1e-4, fused=True)
cm = autosp.compile(m)
ids = torch.randint(0, cfg.vocab, (1, 32769), device="cuda")


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
ev = sorted([(e.time_range.start, e.time_range.end, e.name) for e in prof.events()
             if e.device_type == torch.autograd.DeviceType.CUDA and "Memcpy" not in e.name
             and "Memset" not in e.name], key=lambda x: x[0])
busy = sum(b - a for a, b, _ in ev)
span = ev[-1][1] - ev[0][0]
gaps = []
for (a0, b0, n0), (a1, b1, n1) in zip(ev, ev[1:]):
    g = a1 - max(b0, a0)
    if g > 0:
        gaps.append((g, n0[:60], n1[:60]))
gaps.sort(reverse=True)
print(f"kernels {len(ev)}  span {span/1e3:.1f} ms  busy {busy/1e3:.1f} ms  idle {(span-busy)/1e3:.1f} ms "
      f"({(span-busy)/span*100:.1f} %), gaps > 20us: {sum(1 for g in gaps if g[0] > 20)}")
for g, a, b in gaps[:15]:
    print(f"  {g/1e3:7.3f} ms  after {a}  before {b}")
