import sys, torch
sys.path.insert(0, "/root/repo")
import paper_2604_27089_b200 as autosp
from paper_2604_27089_b200.workloads import CONFIGS, LlamaConfig, LlamaDecoder, lm_loss
cfg = CONFIGS["llama3-8b"]
cfg = LlamaConfig(cfg.name, cfg.d_model, 2, cfg.hq, cfg.hkv, cfg.d_ffn, cfg.vocab)
autosp.reg_passes(["auto_sp", "sp_ac"])
autosp.dist.init(1)
m = LlamaDecoder(cfg, dtype=torch.bfloat16, device="cuda")
cm = autosp.compile(m)
ids = torch.randint(0, cfg.vocab, (1, 32769), device="cuda")
h = cm(ids[:, :-1]); torch.cuda.synchronize(); print("fwd ok", flush=True)
loss = lm_loss(h, m.lm_head, ids[:, 1:]); torch.cuda.synchronize(); print("loss ok", flush=True)
loss.backward(); torch.cuda.synchronize(); print("bwd ok", flush=True)
