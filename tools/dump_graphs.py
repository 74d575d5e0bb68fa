"""Print the AOTAutograd forward / backward graphs (after auto_sp + sp_ac) of a small
Llama-shaped model -- to see which ATen ops surround the AutoSP kernels."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2604_27089_b200 as autosp
from paper_2604_27089_b200 import compiler
from paper_2604_27089_b200.workloads import LlamaConfig, LlamaDecoder, lm_loss

mode = sys.argv[1] if len(sys.argv) > 1 else "auto"
graphs = []


def show(gm, example_inputs):
    graphs.append(gm)
    print(f"==== graph {len(graphs) - 1}\n{gm.code}", flush=True)

    def run(args):
        return gm.forward(*args)
    run._boxed_call = True
    return run


compiler._COMPILER_OVERRIDE = show
autosp.reg_passes(["auto_sp", "sp_ac"], ac_mode=mode)
autosp.dist.init(1)
cfg = LlamaConfig("t", 2048, 1, 32, 8, 8192, vocab=1024)
m = LlamaDecoder(cfg, dtype=torch.bfloat16, device="cuda")
cm = autosp.compile(m)
ids = torch.randint(0, cfg.vocab, (1, 4097), device="cuda")
loss = lm_loss(cm(ids[:, :-1]), m.lm_head, ids[:, 1:])
loss.backward()
torch.cuda.synchronize()
