"""Where does a training step's memory go?  Runs ONE step of a Llama-shaped model
through the AutoSP compile path with the forward/backward GraphModules executed by a
tracing fx.Interpreter (values freed after last use, like the generated code) that
records torch.cuda.memory_allocated() after every node, then prints the peak node of
each graph and the largest live values at that point.

  python tools/mem_trace.py --model llama3-8b --seq 131072 --layers 4 [--ac-mode seq-aware]
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import torch
import torch.fx as fx

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


class MemInterp(fx.Interpreter):
    def __init__(self, gm, tag, log):
        super().__init__(gm, garbage_collect_values=True)
        self.tag, self.log = tag, log
        self.peak = (0, None, [])

    def run_node(self, n):
        try:
            out = super().run_node(n)
        except torch.OutOfMemoryError:
            seen, uniq = set(), []
            for k, v in self.env.items():  # one entry per storage (views share theirs)
                if isinstance(v, torch.Tensor) and v.is_cuda:
                    sid = v.untyped_storage().data_ptr()
                    if sid not in seen:
                        seen.add(sid)
                        uniq.append((v.untyped_storage().nbytes(), k.name, str(k.target),
                                     tuple(v.shape)))
            live = sorted(uniq, reverse=True)
            tot = sum(b for b, *_ in live)
            print(json.dumps({"oom_in": self.tag, "at": n.name, "target": str(n.target),
                              "allocated_gb": torch.cuda.memory_allocated() / 1e9,
                              "env_live_gb": tot / 1e9, "n_live": len(live),
                              "live_top": [(round(b / 1e9, 3), nm, t, sh) for b, nm, t, sh in live[:40]]}),
                  flush=True)
            raise
        a = torch.cuda.memory_allocated()
        if a > self.peak[0]:
            live = []
            for k, v in self.env.items():
                if isinstance(v, torch.Tensor) and v.is_cuda:
                    live.append((v.untyped_storage().nbytes(), k.name, str(k.target), tuple(v.shape)))
            if isinstance(out, torch.Tensor):
                live.append((out.untyped_storage().nbytes(), n.name, str(n.target), tuple(out.shape)))
            live.sort(reverse=True)
            self.peak = (a, n.name, live[:25])
        return out

    def report(self):
        a, name, live = self.peak
        self.log.append({"graph": self.tag, "peak_gb": a / 1e9, "at": name,
                         "live_top": [(round(b / 1e9, 3), nm, t, sh) for b, nm, t, sh in live]})


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama3-8b")
    ap.add_argument("--seq", type=int, default=131072)
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--ac-mode", default="seq-aware")
    ap.add_argument("--reserve-gb", type=float, default=0.0,
                    help="allocate this much first (e.g. 32 = the bf16 AdamW moments of the 8B "
                         "shape, present from the second step on)")
    a = ap.parse_args()
    reserve = torch.empty(int(a.reserve_gb * 1e9), dtype=torch.uint8, device="cuda") \
        if a.reserve_gb else None  # noqa: F841 (held for the whole step)
    import paper_2604_27089_b200 as autosp
    from paper_2604_27089_b200 import compiler, sp_ac
    from paper_2604_27089_b200.workloads import CONFIGS, LlamaConfig, LlamaDecoder, lm_loss
    cfg = CONFIGS[a.model]
    cfg = LlamaConfig(cfg.name, cfg.d_model, a.layers, cfg.hq, cfg.hkv, cfg.d_ffn, cfg.vocab)
    log: list = []
    interps = []

    def traced_compiler(gm, example_inputs):
        tag = f"graph{len(interps)}"

        def run(args):
            it = MemInterp(gm, tag, log)
            interps.append(it)
            out = it.run(*args)
            it.report()
            return out
        run._boxed_call = True
        return run

    compiler._COMPILER_OVERRIDE = traced_compiler
    autosp.reg_passes(["auto_sp", "sp_ac"], ac_mode=a.ac_mode)
    autosp.dist.init(1)
    m = LlamaDecoder(cfg, dtype=torch.bfloat16, device="cuda")
    cm = autosp.compile(m)
    ids = torch.randint(0, cfg.vocab, (1, a.seq + 1), device="cuda")
    base = torch.cuda.memory_allocated()
    hidden = cm(ids[:, :-1])
    after_fwd = torch.cuda.memory_allocated()
    print(json.dumps({"after_fwd_gb": after_fwd / 1e9,
                      "plan": {k: v for k, v in sp_ac.LAST_PLAN.items()
                               if k not in ("saved", "saved_detail", "bw_recomputed_ops")}}), flush=True)
    for d in sp_ac.LAST_PLAN.get("saved_detail", []):
        if "primals" not in d[0] and not d[1].endswith("::t"):
            print("saved", d, flush=True)
    loss = lm_loss(hidden, m.lm_head, ids[:, 1:])
    print(json.dumps({"after_loss_gb": torch.cuda.memory_allocated() / 1e9,
                      "peak_so_far_gb": torch.cuda.max_memory_allocated() / 1e9}), flush=True)
    del hidden
    loss.backward()
    torch.cuda.synchronize()
    print(json.dumps({"static_gb": base / 1e9, "after_fwd_gb": after_fwd / 1e9,
                      "peak_gb": torch.cuda.max_memory_allocated() / 1e9,
                      "plan": {k: v for k, v in sp_ac.LAST_PLAN.items() if k not in ("saved", "saved_detail")}}))
    for d in sp_ac.LAST_PLAN.get("saved_detail", []):
        if "primals" not in d[0] and not d[1].endswith("::t"):
            print("saved", d)
    for r in log:
        print(json.dumps(r))


if __name__ == "__main__":
    main()
