"""Maximum trainable context (BASELINE.json configs[3]: Llama-3-8B shape, OOM frontier)
on the GPUs of this launch: runs one full training step (fwd + bwd + AdamW) per
candidate sequence length in a FRESH process (an OOM must not poison the next probe) and
reports the largest length that completes, with peak memory and step time.

  python tools/max_context.py --model llama3-8b --seqs 32768,65536,98304,131072 [--no-sp-ac]
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def probe(model: str, seq: int, sp_ac: bool, layers: int | None, opt: str = "torch") -> dict:
    code = f"""
import sys, time, json, torch
sys.path.insert(0, {str(ROOT)!r})
import paper_2604_27089_b200 as autosp
from paper_2604_27089_b200.workloads import CONFIGS, LlamaConfig, LlamaDecoder, lm_loss
cfg = CONFIGS[{model!r}]
if {layers!r}:
    cfg = LlamaConfig(cfg.name, cfg.d_model, {layers!r}, cfg.hq, cfg.hkv, cfg.d_ffn, cfg.vocab)
autosp.reg_passes({['auto_sp', 'sp_ac'] if sp_ac else ['auto_sp']!r})
autosp.dist.init(1)
torch.manual_seed(0)
m = LlamaDecoder(cfg, dtype=torch.bfloat16, device='cuda')
if {opt!r} == "torch":
    opt = torch.optim.AdamW(m.parameters(), lr=1e-4, fused=True)
    cm = autosp.compile(m)
else:  # the bf16 multi-tensor kernel; "in-backward": updates inside the compiled backward
    from paper_2604_27089_b200.optim import AdamW
    opt = AdamW(m.parameters(), lr=1e-4)
    cm = autosp.compile(m, optimizer=opt if {opt!r} == "in-backward" else None)
ids = torch.randint(0, cfg.vocab, (1, {seq} + 1), device='cuda')
t0 = None
from paper_2604_27089_b200 import sp_ac
phase = "init"
gb = lambda: round(torch.cuda.memory_allocated() / 1e9, 2)
marks = {{"static_gb": gb()}}
try:
    for it in range(2):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        phase = "forward"
        hidden = cm(ids[:, :-1])
        marks["after_fwd_gb"] = gb(); marks["fwd_peak_gb"] = round(torch.cuda.max_memory_allocated() / 1e9, 2)
        phase = "loss"
        loss = lm_loss(hidden, m.lm_head, ids[:, 1:])
        del hidden
        phase = "backward"
        loss.backward()
        marks["after_bwd_gb"] = gb()
        phase = "optimizer"
        opt.step(); opt.zero_grad(set_to_none=True)
        torch.cuda.synchronize()
except torch.OutOfMemoryError as e:
    msg = str(e).split("\\n")[0]
    pl = sp_ac.LAST_PLAN
    print(json.dumps({{"ok": False, "oom": True, "phase": phase, "iter": it, "error": msg[:400],
                      "marks": marks, "peak_gb": torch.cuda.max_memory_allocated() / 1e9,
                      "ac_applied": pl.get("mode_applied"), "n_saved": len(pl.get("saved", [])),
                      "saved_gb": pl.get("cut_bytes", 0) / 1e9}}))
    sys.exit(3)
pl = sp_ac.LAST_PLAN
print(json.dumps({{"ok": True, "step_s": time.perf_counter() - t0, "marks": marks,
                  "peak_gb": torch.cuda.max_memory_allocated() / 1e9, "loss": float(loss),
                  "ac_applied": pl.get("mode_applied"), "saved_gb": pl.get("cut_bytes", pl.get("save_all_bytes", 0)) / 1e9}}))
"""
    t0 = time.time()
    env = dict(os.environ, PYTORCH_CUDA_ALLOC_CONF="expandable_segments:True")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                       timeout=3600, env=env)
    out = {"seq": seq, "sp_ac": sp_ac, "opt": opt, "wall_s": round(time.time() - t0, 1)}
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    if lines:
        out.update(json.loads(lines[-1]))
    else:
        err = (r.stderr or "").strip()
        tail = [l for l in err.splitlines() if l.strip()]
        out.update(ok=False, oom="out of memory" in err.lower() or "OutOfMemory" in err,
                   error=(tail[-1][-300:] if tail else f"rc={r.returncode}"))
    print(json.dumps(out), flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama3-8b")
    ap.add_argument("--seqs", default="32768,65536,98304,131072")
    ap.add_argument("--no-sp-ac", action="store_true")
    ap.add_argument("--layers", type=int, default=None)
    ap.add_argument("--opt", default="torch", choices=["torch", "autosp", "in-backward"],
                    help="optimizer: torch fused AdamW, the autosp bf16 AdamW kernel, or that "
                         "kernel applied inside the compiled backward (gradients never all live)")
    a = ap.parse_args()
    res = [probe(a.model, int(s), not a.no_sp_ac, a.layers, a.opt) for s in a.seqs.split(",")]
    ok = [r["seq"] for r in res if r.get("ok")]
    print(json.dumps({"model": a.model, "sp_ac": not a.no_sp_ac, "opt": a.opt, "n_gpus": 1,
                      "max_trainable_seq": max(ok) if ok else None, "probes": res}))


if __name__ == "__main__":
    main()
