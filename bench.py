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
class CpuSampledStep:
    """The reference's CPU path (the oracle port: NumPy/OpenBLAS fp32 on all host
    threads, attention by the reference's recipe executor.py:132-142 / autodiff.py:156-214)
    EXECUTING a bounded sample of the same training step: `blocks` runs of `block`
    consecutive query tokens at stratified positions t_i = (i + 1/2)·S/blocks of the
    S-token sequence go through the whole model depth, forward and backward -- every
    layer's norms, projections, SwiGLU MLP and the LM head + cross entropy on those
    tokens, and each block's attention rows against their FULL causal prefix of t_i
    keys/values (all q heads, GQA; the reference's score-matrix recipe on a [block, t_i]
    slab) -- so the work per sampled token averages the real step's per-token work (mean
    prefix S/2).
    Not included: the K/V projections of the prefix tokens (each is the sampled-token
    projection work of another token), and the optimizer step (per step, not per token:
    its share of a 32K-token step is < 0.01 %).  One layer's weights serve every layer
    (the same GEMM shapes; 240 MB per layer streams from DRAM either way)."""

    def __init__(self, cfg, S: int, blocks: int = 1, block: int = 4, seed: int = 0):
        import numpy as np
        self.np = np
        n_tok = blocks * block
        self.cfg, self.S, self.n, self.block = cfg, S, n_tok, block
        rng = np.random.default_rng(seed)
        f32 = np.float32
        d, dm = cfg.head_dim, cfg.d_model
        w = lambda *sh: ((rng.random(sh, dtype=f32) - f32(0.5)) * f32(0.04))
        self.wqkv = w((cfg.hq + 2 * cfg.hkv) * d, dm)
        self.wo = w(dm, cfg.hq * d)
        self.w13 = w(2 * cfg.d_ffn, dm)
        self.w2 = w(dm, cfg.d_ffn)
        self.wlm = w(cfg.vocab, dm)
        self.g1 = np.ones(dm, f32)
        self.g2 = np.ones(dm, f32)
        self.kbuf = rng.standard_normal((1, S, cfg.hkv, d), dtype=f32)
        self.vbuf = rng.standard_normal((1, S, cfg.hkv, d), dtype=f32)
        self.x0 = rng.standard_normal((n_tok, dm), dtype=f32)
        self.labels = rng.integers(0, cfg.vocab, n_tok)
        # last query position of each block (the block attends keys [0, t])
        self.pos = [min(S - 1, int((i + 0.5) * S / blocks) + block - 1) for i in range(blocks)]

    def run(self) -> float:
        from oracle import seqcomp_oracle as orc
        np, cfg, n = self.np, self.cfg, self.n
        d, hq = cfg.head_dim, cfg.hq
        t0 = time.perf_counter()
        x, caches = self.x0, []
        for _ in range(cfg.layers):
            h1 = orc.rmsnorm(x, self.g1)
            q = (h1 @ self.wqkv.T)[:, :hq * d].reshape(n, hq, d)
            o = np.empty_like(q)
            B = self.block
            for i, t in enumerate(self.pos):
                o[i * B:(i + 1) * B] = orc.attention_fwd(
                    q[None, i * B:(i + 1) * B], self.kbuf[:, :t + 1], self.vbuf[:, :t + 1],
                    causal=False)[0][0]
            xm = x + o.reshape(n, hq * d) @ self.wo.T
            h2 = orc.rmsnorm(xm, self.g2)
            gu = h2 @ self.w13.T
            gt, up = gu[:, :cfg.d_ffn], gu[:, cfg.d_ffn:]
            a = orc.silu(gt) * up
            caches.append((x, h1, q, o, xm, h2, gt, up, a))
            x = xm + a @ self.w2.T
        hf = orc.rmsnorm(x, self.g1)
        logits = hf @ self.wlm.T
        p = np.exp(logits - logits.max(-1, keepdims=True))
        p /= p.sum(-1, keepdims=True)
        p[np.arange(n), self.labels] -= 1.0
        _dwlm = p.T @ hf
        dx = orc.rmsnorm_dx(x, self.g1, p @ self.wlm)
        for (xi, h1, q, o, xm, h2, gt, up, a) in reversed(caches):
            _dw2 = dx.T @ a
            da = dx @ self.w2
            dgu = np.concatenate([orc.silu_dx(gt, da * up), da * orc.silu(gt)], axis=1)
            _dw13 = dgu.T @ h2
            dxm = dx + orc.rmsnorm_dx(xm, self.g2, dgu @ self.w13)
            _dg2 = orc.rmsnorm_dw(xm, self.g2, dgu @ self.w13)
            _dwo = dxm.T @ o.reshape(n, hq * d)
            do = (dxm @ self.wo).reshape(n, hq, d)
            dq = np.empty_like(q)
            for i, t in enumerate(self.pos):
                sl = slice(i * B, (i + 1) * B)
                dq[sl] = orc.attention_bwd(q[None, sl], self.kbuf[:, :t + 1],
                                           self.vbuf[:, :t + 1], do[None, sl], causal=False)[0][0]
            dqkv = np.zeros((n, self.wqkv.shape[0]), np.float32)
            dqkv[:, :hq * d] = dq.reshape(n, hq * d)
            _dwqkv = dqkv.T @ h1
            dx = dxm + orc.rmsnorm_dx(xi, self.g1, dqkv @ self.wqkv)
        return time.perf_counter() - t0


def _attention_extrapolated(cfg, b: int, s: int, budget_s: float = 6.0) -> dict:
    """BASELINE.md §3 'attention': the oracle attention fwd+bwd on one head at 2048 tokens,
    its FLOP rate applied to the step's attention FLOPs (labelled extrapolated)."""
    import numpy as np

    from oracle import seqcomp_oracle as orc
    from paper_2604_27089_b200.kernels import causal_attn_flops
    rng = np.random.default_rng(0)
    s_a, d = 2048, cfg.head_dim
    q, k, v, do = (rng.standard_normal((1, s_a, 1, d)).astype(np.float32) for _ in range(4))
    t0, n = time.perf_counter(), 0
    while n == 0 or time.perf_counter() - t0 < budget_s:
        orc.attention_fwd(q, k, v)
        orc.attention_bwd(q, k, v, do)
        n += 1
    rate = 3.5 * causal_attn_flops(1, 1, s_a, d) / ((time.perf_counter() - t0) / n)
    att_total = 3.5 * cfg.layers * causal_attn_flops(b, cfg.hq, s, d)
    return {"gflops": rate / 1e9, "sample": f"1 head x {s_a} tokens fp32, {n} reps",
            "attention_seconds_per_step_extrapolated": att_total / rate}


def _c1_end_to_end() -> dict:
    """BASELINE.md §3 'end-to-end': the oracle's restatement of execute_ranks on the SP
    joint graph (executor.py:344-352) for configs[0] (s 1024, h 8, d 32, d_ffn 1024, L 2,
    P 2), forward + backward, fp32 and fp64 -> tokens/s (measured, not scaled)."""
    import numpy as np

    from oracle import seqcomp_oracle as orc
    dims = orc.Dims(1, 1024, 8, 32, 1024, 2)
    ids, params = orc.random_leaves(dims, 0)
    out = {}
    for name, dt in (("fp32", np.float32), ("fp64", np.float64)):
        orc.sp_forward_backward(dims, ids, params, 2, dtype=dt)
        t0 = time.perf_counter()
        orc.sp_forward_backward(dims, ids, params, 2, dtype=dt)
        out[name] = dims.s / (time.perf_counter() - t0)
    return {"tokens_per_s": out, "config": "configs[0]: s 1024, d_model 256, 8 heads, L 2, P 2"}


def _a2a_gbs() -> dict:
    """BASELINE.md §3 'per-op': the oracle's all_to_all_shards (executor.py:203-230) at
    the per-layer Q shapes of configs[1] (Llama-1B 32K) and configs[2] (Llama-8B 128K),
    P = 8, bf16 payload as uint16, all ranks in one process -> GB/s copied."""
    import numpy as np

    from oracle import seqcomp_oracle as orc
    out = {}
    for name, s, d in (("llama3.2-1b_32k_p8", 32768, 64), ("llama3-8b_128k_p8", 131072, 128)):
        shards = [np.full((1, s // 8, 32, d), j, np.uint16) for j in range(8)]
        orc.all_to_all_shards("seq_to_head", shards)
        t0 = time.perf_counter()
        orc.all_to_all_shards("seq_to_head", shards)
        out[name] = sum(x.nbytes for x in shards) / (time.perf_counter() - t0) / 1e9
    return out


def cpu_baseline(cfg, b: int, s: int, steps: int = 2, warmup: int = 1, blocks: int = 1,
                 block: int = 4, extras: bool = True) -> dict:
    """Measured CPU baseline (see CpuSampledStep): tokens/s = sampled tokens / measured
    seconds per sampled step, plus the BASELINE.md §3 figures."""
    smp = CpuSampledStep(cfg, s, blocks, block)
    n_tok = smp.n
    times = [smp.run() for _ in range(warmup + steps)][warmup:]
    t = statistics.median(times)
    out = {"value": b * n_tok / t, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
           "sample": (f"{n_tok} query tokens per step ({blocks} runs of {block} consecutive "
                      f"tokens at stratified positions of the {s}-token sequence), full depth ({cfg.layers} layers) fwd+bwd + LM head, each "
                      f"attending its full causal prefix (mean {s // 2}); NumPy fp32, "
                      f"OPENBLAS_NUM_THREADS={os.environ.get('OPENBLAS_NUM_THREADS', 'unset')}; "
                      f"optimizer step excluded"),
           "seconds_per_sampled_step": t, "sampled_step_times": times,
           "tokens_per_step": b * n_tok}
    if extras:
        att = _attention_extrapolated(cfg, b, s)
        out["baseline_md_s3"] = {"c1_end_to_end": _c1_end_to_end(), "a2a_gbs": _a2a_gbs(),
                                 "attention_extrapolated": att}
    return out


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from paper_2604_27089_b200.workloads import CONFIGS
    cfg = CONFIGS[args.model]
    r = cpu_baseline(cfg, args.batch, args.seq, steps=args.steps, warmup=args.warmup)
    v = r["value"]
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": r["seconds_per_sampled_step"] * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": (f"{cfg.name} seq {args.seq}: CPU oracle port executing a "
                                    f"bounded sample of the step ({r['sample']})"),
                       "model": cfg.name, "global_batch": args.batch, "seq_len": args.seq,
                       "tokens_per_step": r["tokens_per_step"], "parallelism": "cpu"},
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
    ap.add_argument("--no-sp-ac-block", action="store_true",
                    help="skip the extra seq-aware-vs-save-all comparison steps")
    ap.add_argument("--zero1", default="auto", choices=["auto", "on", "off"],
                    help="N > 1: ZeRO-1 (AdamW state sharded over the SP group, updated "
                         "parameters all-gathered) -- auto: only when the replicated bf16 "
                         "AdamW state would exceed 10 %% of device memory (the in-graph "
                         "gradient all-reduce already overlaps the backward; ZeRO-1 adds an "
                         "exposed all-gather, so it is a memory, not a speed, option)")
    ap.add_argument("--no-zero1", action="store_true", help="same as --zero1 off")
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
    if args.no_zero1:
        args.zero1 = "off"
    opt_state = 2 * 2 * cfg.n_params()  # bf16 first + second moments
    zero1 = P > 1 and (args.zero1 == "on" or (
        args.zero1 == "auto" and opt_state > 0.10 * torch.cuda.get_device_properties(dev).total_memory))
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

    def step(ids_, labels_, cm_=None):
        hidden = (cm if cm_ is None else cm_)(ids_)
        loss = lm_loss(hidden, model.lm_head, labels_)
        loss.backward()  # (P > 1: the SP-partial gradients are all-reduced in-graph)
        opt.step()
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

    ac_applied = sp_ac.LAST_PLAN.get("mode_applied")

    # ---------------- sp_ac block: the same step with seq-aware recomputation forced,
    # against the planner's choice (paper: SP+AC vs SP-only 1.07x step time, 1.66x
    # trainability) -- step time and steady-state peak memory
    spac = None
    if "sp_ac" in passes and ac_applied == "save-all" and not args.no_sp_ac_block:
        def timed(cm_, n):
            torch.cuda.reset_peak_memory_stats(dev)
            barrier()
            a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(n):
                step(ids, labels, cm_)
            z.record()
            barrier()
            ms = torch.tensor([a.elapsed_time(z) / n, torch.cuda.max_memory_allocated(dev)],
                              dtype=torch.float64, device=dev)
            if world > 1:
                tdist.all_reduce(ms, op=tdist.ReduceOp.MAX)
            return float(ms[0]), float(ms[1])
        base_ms, base_mem = timed(cm, 2)
        cm_sa = autosp.compile(model, ac_mode="seq-aware")
        step(ids, labels, cm_sa)  # compile + warm-up
        plan = dict(sp_ac.LAST_PLAN)
        sa_ms, sa_mem = timed(cm_sa, 2)
        spac = {"mode": plan.get("mode_applied"), "ms_per_step": sa_ms,
                "save_all_ms_per_step": base_ms, "step_time_ratio": sa_ms / base_ms,
                "peak_mem_gb": sa_mem / 1e9, "save_all_peak_mem_gb": base_mem / 1e9,
                "peak_mem_ratio": base_mem / sa_mem,
                "saved_bytes_per_rank_gb": (plan.get("saved_bytes") or 0) / 1e9,
                "recomputed_fw_nodes": len(plan.get("recomputed_fw_nodes") or []),
                "paper": "SP+AC vs SP-only: 7 % slower, 1.66x trainability (PAPER.md:321)"}

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
    a2a = None
    if "a2a" in ksum and P > 1:
        v = ksum["a2a"]
        a2a = {"kernel": "standalone reshard launches (handshake + push; per layer the "
                         "dO + delta reshard of the backward).  The q/k/v push runs in K0's "
                         "epilogue, O in K3's, dq/dk/dv in K4's: not separately timed",
               "calls_per_step": v["calls"] / args.steps,
               "bytes_per_call": v["bytes"] / max(v["calls"], 1),
               "us_per_call": v["ms"] * 1e3 / max(v["calls"], 1),
               "gbs": v["bytes"] / (v["ms"] / 1e3) / 1e9 if v["ms"] else None,
               "peak_gbs": 900.0, "peak_kind": "NVLink 5 per direction per GPU (nominal)"}
        a2a["frac"] = a2a["gbs"] / 900.0 if a2a["gbs"] else None
        if os.environ.get("AUTOSP_BENCH_BACKEND") == "gloo":
            a2a["note"] = "ranks share ONE GPU (test harness): loopback, not NVLink"
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
                   "ac_applied": ac_applied,
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
        "a2a": a2a,
        "sp_ac": spac,
        "peak_mem_gb": peak_mem / 1e9,
        "final_loss": loss_v,
        "clocks": clk.summary(),
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, b, S)
    print(json.dumps(line), flush=True)
    if world > 1:
        tdist.barrier()
    return 0


if __name__ == "__main__":
    sys.exit(main())
