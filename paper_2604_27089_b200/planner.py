"""Trainability planner: per-rank memory of one training step of a Llama-shaped model
under Ulysses SP (auto_sp + sp_ac seq-aware + ZeRO-1) and the largest trainable global
sequence it implies (the reference's counterpart is the analytical
``max_trainable_seq`` / ``memory_at``, cost_model.py:152-194, which models fp32 and
unfused O(s^2) attention -- this one models what THIS implementation keeps).

Per rank, with S the global sequence, P the SP size, e = 2 (bf16), L layers:

  static     params + grads (e each) + optimizer state: AdamW moments (2e) and, under
             ZeRO-1 (P > 1), the owned fp shard copy, both divided by P
  saved      what sp_ac keeps per layer in the caching allocator:
               P == 1: x_in [S, d] + O [S, hq*hd] + LSE / rstd
               P  > 1: x_in [S/P, d] + LSE [hq/P, S] fp32 + rstd
  pool       (P > 1) the symmetric receive heap (dist.SymmetricPool, grows on demand):
             the a2a outputs sp_ac keeps per layer -- q/k/v head shards
             [S, (hq + 2 hkv)/P * hd] and the token-major O [S/P, hq*hd] (no head-major O:
             delta = rowsum(dO*O) is formed token-side) -- plus one layer's backward
             reshards (dO head shard, delta, the packed dq/dk/dv gradient)
  transient  the largest backward working set of one layer: the recomputed MLP chunk
             (gate/up and their gradients, chunked at MLP_CHUNK tokens), the attention
             backward's fp32 dQ accumulator and bf16 dq/dk/dv, the recomputed projections,
             plus the LM-head chunk (logits + its gradient pieces)

Calibrated against the measured single-GPU frontier (profiles/max_context_r01_*): the
model is a prediction for P > 1, reported as such."""

from __future__ import annotations

from dataclasses import dataclass

from .workloads import MLP_CHUNK, MLP_CHUNK_TOKENS, LlamaConfig

GB = 1e9
USABLE_FRACTION = 0.97   # of device memory the caching allocator can hand out
CE_CHUNK = 4096          # lm_loss chunk (tokens)


@dataclass
class MemoryEstimate:
    static: float
    saved: float
    transient: float
    pool: float = 0.0

    @property
    def total(self) -> float:
        return self.static + self.saved + self.pool + self.transient


ALIGN = 1024  # dist.SymmetricPool.ALIGN


def _al(n: int) -> int:
    return (n + ALIGN - 1) // ALIGN * ALIGN


def pool_layer_bytes(cfg: LlamaConfig, S: int, P: int, e: int = 2) -> tuple[int, int]:
    """(kept, backward-transient) symmetric-heap bytes of ONE layer at P > 1, slab sizes
    exactly as ops.py allocates them: the q/k/v reshard (one slab of three pieces), the
    token-major O push; in backward the dO and delta reshards and the packed gradient."""
    hd, hq, hkv, sl = cfg.head_dim, cfg.hq, cfg.hkv, S // P
    qkv = _al(_al(e * S * hq // P * hd) + 2 * _al(e * S * hkv // P * hd))
    o_tok = _al(e * sl * hq * hd)
    bwd = _al(e * S * hq // P * hd) + _al(4 * S * hq // P) + _al(e * sl * (hq + 2 * hkv) * hd)
    return qkv + o_tok, bwd


def pool_bytes(cfg: LlamaConfig, S: int, P: int, e: int = 2) -> int:
    """Steady-state high water of the symmetric receive heap of one rank for a training
    step (every layer's kept a2a outputs + one layer's backward reshards); pass it to
    dist.init(pool_bytes=...) to get the whole heap as one segment."""
    if P == 1:
        return 0
    kept, bwd = pool_layer_bytes(cfg, S, P, e)
    return cfg.layers * kept + bwd


def step_memory(cfg: LlamaConfig, S: int, P: int = 1, zero1: bool = True,
                e: int = 2) -> MemoryEstimate:
    d, hd, hq, hkv, L, F = cfg.d_model, cfg.head_dim, cfg.hq, cfg.hkv, cfg.layers, cfg.d_ffn
    n = cfg.n_params()
    opt = 2 * e * n + (e * n if (zero1 and P > 1) else 0)   # moments (+ owned shard copy)
    static = 2 * e * n + (opt / P if (zero1 and P > 1) else 2 * e * n)
    sl = S // P
    if P == 1:
        per_layer = e * sl * (d + hq * hd) + 4 * sl * (hq + 2)          # x_in, O, LSE, rstd
    else:
        per_layer = e * sl * d + 4 * S * hq // P + 4 * sl * 2            # x_in, LSE, rstd
    saved = L * per_layer + e * sl * d                                   # + final hidden
    pool = pool_bytes(cfg, S, P, e)                                      # a2a outputs
    chunk = sl if sl <= MLP_CHUNK else MLP_CHUNK_TOKENS
    mlp = e * chunk * (2 * F) * 2 + e * chunk * F * 2                    # gate/up (+grad), act (+grad)
    dq_acc = 4 * S * hq // P * hd                                        # fp32 dQ accumulator,
    groups = max(hkv // P, 1)                                            # run per kv-head group
    while groups > 1 and dq_acc > (1 << 30):                             # above 1 GiB
        dq_acc //= 2                                                     # (kernels.attn_bwd)
        groups //= 2
    attn = dq_acc + e * S * (hq + 2 * hkv) // P * hd                     # + dq/dk/dv
    if P == 1:
        attn += e * S * hq * hd                                          # dO (in the heap at P > 1)
    proj = e * sl * ((hq + 2 * hkv) * hd + 3 * d)                        # recomputed qkv, x_mid, grads
    head = e * CE_CHUNK * cfg.vocab * 2 + e * cfg.vocab * d + e * sl * d  # logits, dW, dh
    transient = max(mlp, attn) + proj + head
    return MemoryEstimate(static, saved, transient, pool)


def predict_max_context(cfg: LlamaConfig, P: int, device_bytes: float,
                        granule: int | None = None, zero1: bool = True) -> int:
    """Largest S (a multiple of `granule`, default 16 * 128 * P) whose estimate fits."""
    granule = granule or 16 * 128 * P
    budget = USABLE_FRACTION * device_bytes
    lo, hi = 0, granule
    while step_memory(cfg, hi, P, zero1).total <= budget:
        lo, hi = hi, hi * 2
        if hi > 1 << 26:
            break
    while hi - lo > granule:
        mid = (lo + hi) // 2 // granule * granule
        if mid <= lo:
            break
        if step_memory(cfg, mid, P, zero1).total <= budget:
            lo = mid
        else:
            hi = mid
    return lo
