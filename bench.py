#!/usr/bin/env python
"""Training throughput of the AutoSP Ulysses-SP hot path on B200 (BASELINE.json metric:
"train tokens/s and max trainable seq len at 1/2/4/8 B200 (Ulysses SP)").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl autosp|reference]
  python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N ...

Workload (BASELINE.json configs[1]): Llama-3.2-1B-shaped synthetic decoder, global
sequence 32K tokens, batch 1, bf16, Ulysses SP over all N GPUs (P = N; strong scaling:
the 32K-token step is split across the ranks), auto_sp + sp_ac, AdamW.  One step =
forward + backward + SP-group gradient reduction + optimizer step on one batch.

Prints ONE JSON line (rank 0).  `value` is device-timed (CUDA events, max over ranks)
with inputs resident; `e2e` goes through the public API with the token ids copied from
pinned host memory and the loss read back every step.  `roofline` is the dominant
kernel (attention backward) measured live with CUDA events; `cpu_baseline` times the
CPU oracle (a restatement of the reference's NumPy path) on a bounded sample.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "train tokens/s (Ulysses SP)"
UNIT = "tokens/s"


def _peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text()), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, \
            "fallback"


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            parts = [p.strip() for p in l.split(",")]
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except (ValueError, IndexError):
                continue
            for n, v in zip(names, parts[3:]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------- CPU baseline
def cpu_oracle_sample(cfg, b: int, s: int, budget_s: float = 12.0) -> dict:
    """Time the CPU oracle (restated reference path, NumPy/OpenBLAS, all host threads)
    on a bounded sample of the SAME step and scale it to tokens/s:
      attention: oracle attention_fwd + attention_bwd on one head at s_a tokens (fp32),
                 rate applied to the step's causal attention FLOPs (fwd 1x + bwd 2.5x);
      dense:     one transformer layer's projections/MLP fwd+bwd (6 * params * tokens)
                 on a 512-token sample, rate applied to all layers + LM head."""
    import numpy as np

    from oracle import seqcomp_oracle as orc
    from paper_2604_27089_b200.kernels import causal_attn_flops

    rng = np.random.default_rng(0)
    d = cfg.head_dim
    s_a = 2048
    q = rng.standard_normal((1, s_a, 1, d)).astype(np.float32)
    k = rng.standard_normal((1, s_a, 1, d)).astype(np.float32)
    v = rng.standard_normal((1, s_a, 1, d)).astype(np.float32)
    do = rng.standard_normal((1, s_a, 1, d)).astype(np.float32)
    t0 = time.perf_counter()
    n_att = 0
    while True:
        orc.attention_fwd(q, k, v)
        orc.attention_bwd(q, k, v, do)
        n_att += 1
        if time.perf_counter() - t0 > budget_s / 2:
            break
    t_att = (time.perf_counter() - t0) / n_att
    rate_att = 3.5 * causal_attn_flops(1, 1, s_a, d) / t_att

    ntok, dm = 512, cfg.d_model
    ws = [rng.standard_normal(sh).astype(np.float32) * 0.02 for sh in
          [((cfg.hq + 2 * cfg.hkv) * d, dm), (dm, cfg.hq * d), (2 * cfg.d_ffn, dm), (dm, cfg.d_ffn)]]
    x = rng.standard_normal((ntok, dm)).astype(np.float32)
    t0 = time.perf_counter()
    n_den = 0
    layer_params = sum(w.size for w in ws)
    while True:
        for w in ws:
            xi = x if w.shape[1] == dm else rng.standard_normal((ntok, w.shape[1])).astype(np.float32)
            y = xi @ w.T
            _ = y @ w          # dX
            _ = y.T @ xi       # dW
        n_den += 1
        if time.perf_counter() - t0 > budget_s / 2:
            break
    t_den = (time.perf_counter() - t0) / n_den
    rate_den = 6.0 * layer_params * ntok / t_den

    att_total = 3.5 * cfg.layers * causal_attn_flops(b, cfg.hq, s, d)
    dense_total = 6.0 * (cfg.n_params() - cfg.vocab * cfg.d_model) * b * s
    t_step = att_total / rate_att + dense_total / rate_den
    return {"value": b * s / t_step, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
            "sample": (f"oracle attention fwd+bwd, 1 head x {s_a} tokens (fp32, {n_att} reps, "
                       f"{rate_att/1e9:.1f} GFLOP/s) + one layer's dense fwd+bwd on {ntok} tokens "
                       f"({rate_den/1e9:.1f} GFLOP/s), scaled by FLOPs to the {s}-token step"),
            "seconds_per_step_extrapolated": t_step}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from paper_2604_27089_b200.workloads import CONFIGS
    cfg = CONFIGS[args.model]
    vals = []
    for i in range(args.warmup + args.steps):
        r = cpu_oracle_sample(cfg, args.batch, args.seq, budget_s=4.0)
        if i >= args.warmup:
            vals.append(r["value"])
    v = statistics.median(vals)
    r["value"] = v
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": args.batch * args.seq / v * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{cfg.name} seq {args.seq} (CPU oracle, bounded sample)",
                       "model": cfg.name, "global_batch": args.batch, "seq_len": args.seq,
                       "parallelism": f"sp{args.gpus}"},
            "cpu_baseline": r,
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- GPU run
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="autosp", choices=["autosp", "reference"])
    ap.add_argument("--model", default="llama3.2-1b")
    ap.add_argument("--seq", type=int, default=32768)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--ac-mode", default="auto",
                    help="sp_ac policy: auto (recompute only if the step would not fit), "
                         "seq-aware, conservative, seq-aware-all")
    ap.add_argument("--no-sp-ac", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-zero1", action="store_true",
                    help="N > 1: all-reduce gradients + replicated AdamW instead of ZeRO-1")
    ap.add_argument("--layers", type=int, default=None, help="override (debug only; invalid bench)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as tdist

    import paper_2604_27089_b200 as autosp
    from paper_2604_27089_b200 import kernels, sp_ac
    from paper_2604_27089_b200.workloads import CONFIGS, LlamaConfig, LlamaDecoder, lm_loss

    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if world > 1:
        # NCCL for real multi-GPU runs; AUTOSP_BENCH_BACKEND=gloo lets several ranks share
        # one GPU to exercise this path (the reshard itself never uses NCCL)
        tdist.init_process_group(os.environ.get("AUTOSP_BENCH_BACKEND", "nccl"))
    rank = tdist.get_rank() if world > 1 else 0
    passes = ["auto_sp"] if args.no_sp_ac else ["auto_sp", "sp_ac"]
    autosp.reg_passes(passes, ac_mode=args.ac_mode)
    cfg = CONFIGS[args.model]
    if args.layers:
        cfg = LlamaConfig(cfg.name + f"-L{args.layers}", cfg.d_model, args.layers, cfg.hq,
                          cfg.hkv, cfg.d_ffn, cfg.vocab)
    P, b, S = world, args.batch, args.seq
    # the symmetric receive heap sized up front from the planner (it would grow on demand)
    from paper_2604_27089_b200.planner import pool_bytes
    st = autosp.dist.init(world, pool_bytes=(int(pool_bytes(cfg, S, P) * b * 1.05) + (64 << 20))
                          if P > 1 else None)
    dev = st.device if st.device.type == "cuda" else torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    if S % P:
        raise SystemExit("seq not divisible by world")
    sl = S // P

    torch.manual_seed(0)
    model = LlamaDecoder(cfg, dtype=torch.bfloat16, device=dev)
    zero1 = P > 1 and not args.no_zero1
    if zero1:  # ZeRO-1 over the SP group: reduce-scatter + sharded AdamW + all-gather
        from paper_2604_27089_b200.zero import ShardedAdamW
        opt = ShardedAdamW(model.parameters(), st, lr=1e-4)
    else:
        from paper_2604_27089_b200.optim import AdamW  # multi-tensor bf16 kernel
        opt = AdamW(model.parameters(), lr=1e-4)
    cm = autosp.compile(model)
    g = torch.Generator(device="cpu").manual_seed(1234)
    ids_full = torch.randint(0, cfg.vocab, (b, S + 1), generator=g)
    ids_host = ids_full[:, rank * sl:(rank + 1) * sl].contiguous().pin_memory()
    lab_host = ids_full[:, rank * sl + 1:(rank + 1) * sl + 1].contiguous().pin_memory()
    ids = ids_host.to(dev)
    labels = lab_host.to(dev)
    params = list(model.parameters())

    def step(ids_, labels_):
        hidden = cm(ids_)
        loss = lm_loss(hidden, model.lm_head, labels_)
        loss.backward()
        if P > 1 and not zero1:
            autosp.dist.reduce_gradients(params, st)
        opt.step()  # (ShardedAdamW reduces the SP-partial gradients itself)
        opt.zero_grad(set_to_none=True)
        return loss

    def barrier():
        if world > 1:
            tdist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step(ids, labels)
    barrier()
    peak_mem = torch.cuda.max_memory_allocated(dev)

    # ---------------- device-timed region (inputs resident)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    kernels.LOG.reset(timing=True)
    barrier()
    with ClockSampler(dev.index or 0) as clk:
        torch.cuda.nvtx.range_push("timed")
        e0.record()
        for _ in range(args.steps):
            loss = step(ids, labels)
        e1.record()
        torch.cuda.nvtx.range_pop()
        barrier()
    launches = kernels.LOG.launches
    ksum = kernels.LOG.summary()
    kernels.LOG.enabled = False
    t_ms = e0.elapsed_time(e1)
    if world > 1:
        tt = torch.tensor([t_ms], device=dev)
        tdist.all_reduce(tt, op=tdist.ReduceOp.MAX)
        t_ms = float(tt)
    value = b * S * args.steps / (t_ms / 1e3)

    # ---------------- end-to-end through the public API (host copies + loss readback)
    ids_dev = torch.empty_like(ids)
    lab_dev = torch.empty_like(labels)
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ids_dev.copy_(ids_host, non_blocking=True)
        lab_dev.copy_(lab_host, non_blocking=True)
        loss_v = float(step(ids_dev, lab_dev).item())
    barrier()
    t_e2e = time.perf_counter() - t0
    if world > 1:
        tt = torch.tensor([t_e2e], device=dev)
        tdist.all_reduce(tt, op=tdist.ReduceOp.MAX)
        t_e2e = float(tt)
    e2e = {"value": b * S * args.steps / t_e2e, "unit": UNIT,
           "h2d_bytes_per_step": (ids_host.numel() + lab_host.numel()) * ids_host.element_size(),
           "d2h_bytes_per_step": 4}

    if rank != 0:
        if world > 1:
            tdist.barrier()
        return 0

    peaks, peak_kind = _peaks()
    sustained = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
    dom = ksum.get("attn_bwd", {"ms": 0.0, "flops": 0.0, "calls": 0})
    achieved = dom["flops"] / (dom["ms"] / 1e3) / 1e12 if dom["ms"] else None
    traffic = None
    try:
        prof = json.loads((ROOT / "profiles" / "roofline_traffic.json").read_text())
        traffic = prof.get(f"{cfg.name}_s{S}_p{P}_attn_bwd_dram_bytes_per_launch")
    except Exception:
        pass
    step_ms = t_ms / args.steps
    kern = {k: {"calls_per_step": v["calls"] / args.steps, "ms_per_step": v["ms"] / args.steps,
                "share_of_step": v["ms"] / t_ms,
                "tflops": (v["flops"] / (v["ms"] / 1e3) / 1e12) if v["ms"] and v["flops"] else None}
            for k, v in ksum.items()}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (random token ids, random-init weights N(0, 0.02^2))",
        "config": {"workload": f"{cfg.name} synthetic, global seq {S}, batch {b}" + (
                       " (BASELINE.json configs[1]; at N=1 the single-GPU case)"
                       if (cfg.name, S) == ("llama3.2-1b", 32768) else ""),
                   "model": cfg.name, "global_batch": b, "seq_len": S,
                   "parallelism": f"sp{P}" + ("+zero1" if zero1 else ""), "passes": passes,
                   "ac_mode": args.ac_mode,
                   "ac_applied": sp_ac.LAST_PLAN.get("mode_applied"),
                   "l2": f"working set (weights {2 * cfg.n_params() / 1e9:.1f} GB + activations)"
                         " >> 126 MB L2; no flush"},
        "e2e": e2e,
        "gpu_launches": launches,
        "roofline": {"kernel": "attn_bwd (K4: pre + tcgen05 main + post, per launch)",
                     "bound": "tensor", "achieved": achieved, "peak": sustained,
                     "unit": "TFLOP/s",
                     "frac": (achieved / sustained) if achieved else None,
                     "peak_kind": f"{peak_kind} bf16 sustained (kernel timed inside a long step)",
                     "algorithmic_flops_per_launch": dom["flops"] / max(dom["calls"], 1),
                     "traffic": traffic},
        "kernels": kern,
        "peak_mem_gb": peak_mem / 1e9,
        "final_loss": loss_v,
        "clocks": clk.summary(),
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_oracle_sample(cfg, b, S)
    print(json.dumps(line), flush=True)
    if world > 1:
        tdist.barrier()
    return 0


if __name__ == "__main__":
    sys.exit(main())
