"""Synthetic user models the AutoSP path is exercised on (plain PyTorch modules: the
auto_sp pass finds their ``scaled_dot_product_attention`` calls and position indices).

* ``SeqcompDecoder`` — the reference's parity model, ``transformer.py:42-113``:
  embed(ids % vocab) + raw position, per layer RMSNorm(1e-6) -> shared qkv Linear ->
  attention with q = k = v -> out Linear -> +res -> RMSNorm -> up Linear -> silu ->
  down Linear -> +res; loss = sum(x^2).  Parameter names match the oracle's.
* ``LlamaDecoder`` — Llama-3-shaped synthetic model for the throughput configs
  (BASELINE.json configs 2-5): fused QKV with GQA, RoPE (theta 5e5), SwiGLU, RMSNorm
  (the fused variant runs the autosp RMSNorm / qkv_rope / swiglu kernels),
  chunked-vocab cross-entropy head outside the compiled body.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass

import torch
import torch.nn as nn
import torch.nn.functional as F

from .auto_sp import positions


def rmsnorm(x: torch.Tensor, w: torch.Tensor, eps: float) -> torch.Tensor:
    """executor.py:43-45, computed in fp32 (or the input precision if wider)."""
    ct = torch.promote_types(x.dtype, torch.float32)
    xf = x.to(ct)
    y = xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + eps)
    return (y * w.to(ct)).to(x.dtype)


# ----------------------------------------------------------------------------- reference model
@dataclass(frozen=True)
class SeqcompDims:
    b: int
    s: int
    h: int
    d: int
    d_ffn: int
    layers: int
    vocab: int = 64

    @property
    def d_model(self) -> int:
        return self.h * self.d


class SeqcompDecoder(nn.Module):
    """transformer.py:42-113 as a torch module (single rank sees its sequence shard)."""

    def __init__(self, dims: SeqcompDims, dtype=torch.float32, device=None):
        super().__init__()
        self.dims = dims
        dm, f = dims.d_model, dims.d_ffn
        mk = lambda *shape: nn.Parameter(torch.zeros(*shape, dtype=dtype, device=device))
        self.embed_table = mk(dims.vocab, dm)
        self.norm1 = nn.ParameterList([mk(dm) for _ in range(dims.layers)])
        self.qkv = nn.ParameterList([mk(dm, dm) for _ in range(dims.layers)])
        self.out = nn.ParameterList([mk(dm, dm) for _ in range(dims.layers)])
        self.norm2 = nn.ParameterList([mk(dm) for _ in range(dims.layers)])
        self.up = nn.ParameterList([mk(f, dm) for _ in range(dims.layers)])
        self.down = nn.ParameterList([mk(dm, f) for _ in range(dims.layers)])

    def named_reference_params(self) -> dict[str, nn.Parameter]:
        out = {"embed_table": self.embed_table}
        for l in range(self.dims.layers):
            out.update({f"l{l}.norm1.w": self.norm1[l], f"l{l}.qkv.w": self.qkv[l],
                        f"l{l}.out.w": self.out[l], f"l{l}.norm2.w": self.norm2[l],
                        f"l{l}.mlp.up.w": self.up[l], f"l{l}.mlp.down.w": self.down[l]})
        return out

    @torch.no_grad()
    def load_reference(self, params: dict) -> None:
        for k, p in self.named_reference_params().items():
            p.copy_(torch.as_tensor(params[k], dtype=p.dtype))

    def forward(self, ids: torch.Tensor):
        dims = self.dims
        b, s = ids.shape
        x = self.embed_table[ids.long() % dims.vocab]                 # executor.py:153-154
        pos = positions(s, device=ids.device).to(x.dtype)             # executor.py:68-70
        x = x + pos.view(s, 1)
        for l in range(dims.layers):
            res = x
            y = rmsnorm(x, self.norm1[l], 1e-6)
            y = y @ self.qkv[l].t()
            y = y.view(b, s, dims.h, dims.d).transpose(1, 2)
            y = F.scaled_dot_product_attention(y, y, y, is_causal=True)   # q = k = v
            y = y.transpose(1, 2).reshape(b, s, dims.d_model)
            x = y @ self.out[l].t() + res
            res = x
            y = rmsnorm(x, self.norm2[l], 1e-6)
            y = F.silu(y @ self.up[l].t())
            x = y @ self.down[l].t() + res
        return x, (x * x).sum()


# ----------------------------------------------------------------------------- Llama shape
@dataclass(frozen=True)
class LlamaConfig:
    name: str
    d_model: int
    layers: int
    hq: int
    hkv: int
    d_ffn: int
    vocab: int = 128256
    rope_theta: float = 500000.0
    eps: float = 1e-5

    @property
    def head_dim(self) -> int:
        return self.d_model // self.hq

    def n_params(self) -> int:
        d, L = self.d_model, self.layers
        qkv = d * (self.hq + 2 * self.hkv) * self.head_dim
        per = qkv + self.hq * self.head_dim * d + 3 * d * self.d_ffn + 2 * d
        return L * per + 2 * self.vocab * d + d


LLAMA_1B = LlamaConfig("llama3.2-1b", 2048, 16, 32, 8, 8192)
LLAMA_8B = LlamaConfig("llama3-8b", 4096, 32, 32, 8, 14336)
CONFIGS = {c.name: c for c in (LLAMA_1B, LLAMA_8B)}


def rope(x: torch.Tensor, cos: torch.Tensor, sin: torch.Tensor) -> torch.Tensor:
    """x [b, s, h, d]; cos/sin [s, d/2] (rotate-half convention)."""
    d2 = x.shape[-1] // 2
    x1, x2 = x[..., :d2], x[..., d2:]
    c = cos.view(1, cos.shape[0], 1, d2).to(x.dtype)
    s_ = sin.view(1, sin.shape[0], 1, d2).to(x.dtype)
    return torch.cat((x1 * c - x2 * s_, x2 * c + x1 * s_), dim=-1)


MLP_CHUNK = 32768  # sequences longer than this run the MLP chunked (memory only) ...
MLP_CHUNK_TOKENS = 16384  # ... in chunks of this many tokens: the backward recomputes one
                          # chunk's [tokens, 2*d_ffn] gate/up at a time at its memory peak
                          # (Llama-3-8B at 224K: 0.94 GB instead of 1.88 GB)
FUSE_RESIDUAL = os.environ.get("AUTOSP_FUSE_RESIDUAL", "1") == "1"  # addmm epilogue adds


class LlamaBlock(nn.Module):
    def __init__(self, cfg: LlamaConfig, dtype, device, fused: bool = True):
        super().__init__()
        d, hd = cfg.d_model, cfg.head_dim
        kw = dict(dtype=dtype, device=device)
        self.cfg = cfg
        self.fused = fused
        self.norm1 = nn.Parameter(torch.ones(d, **kw))
        self.wqkv = nn.Parameter(torch.empty((cfg.hq + 2 * cfg.hkv) * hd, d, **kw))
        self.wo = nn.Parameter(torch.empty(d, cfg.hq * hd, **kw))
        self.norm2 = nn.Parameter(torch.ones(d, **kw))
        self.w13 = nn.Parameter(torch.empty(2 * cfg.d_ffn, d, **kw))
        self.w2 = nn.Parameter(torch.empty(d, cfg.d_ffn, **kw))

    def forward(self, x, cos, sin, pos):
        cfg = self.cfg
        b, s, _ = x.shape
        hd = cfg.head_dim
        if self.fused:
            from . import ops
            h = ops.rms_norm(x, self.norm1, cfg.eps)
            qkv = (h @ self.wqkv.t()).view(b, s, cfg.hq + 2 * cfg.hkv, hd)
            q, k, v = ops.qkv_rope(qkv, pos, cfg.rope_theta, cfg.hq, cfg.hkv)
        else:
            h = rmsnorm(x, self.norm1, cfg.eps)
            qkv = (h @ self.wqkv.t()).view(b, s, cfg.hq + 2 * cfg.hkv, hd)
            q = rope(qkv[:, :, :cfg.hq], cos, sin)
            k = rope(qkv[:, :, cfg.hq:cfg.hq + cfg.hkv], cos, sin)
            v = qkv[:, :, cfg.hq + cfg.hkv:]
        o = F.scaled_dot_product_attention(q.transpose(1, 2), k.transpose(1, 2),
                                           v.transpose(1, 2), is_causal=True, enable_gqa=True)
        if self.fused and FUSE_RESIDUAL:  # residual adds in the GEMM epilogue (beta = 1)
            d = cfg.d_model
            x = torch.addmm(x.reshape(b * s, d), o.transpose(1, 2).reshape(b * s, cfg.hq * hd),
                            self.wo.t()).view(b, s, d)
        else:
            x = x + o.transpose(1, 2).reshape(b, s, cfg.hq * hd) @ self.wo.t()
        if self.fused:
            from . import ops
            h = ops.rms_norm(x, self.norm2, cfg.eps)
            if s <= MLP_CHUNK and FUSE_RESIDUAL:
                return torch.addmm(x.reshape(b * s, d), ops.swiglu(h @ self.w13.t()).view(b * s, -1),
                                   self.w2.t()).view(b, s, d)
            if s <= MLP_CHUNK:
                return x + ops.swiglu(h @ self.w13.t()) @ self.w2.t()
            # long contexts: the MLP in sequence chunks, so its [s, 2*d_ffn] intermediate
            # (and, under sp_ac, its recomputation in backward) is live one chunk at a time
            return x + torch.cat([ops.swiglu(hc @ self.w13.t()) @ self.w2.t()
                                  for hc in h.split(MLP_CHUNK_TOKENS, dim=1)], dim=1)
        h = rmsnorm(x, self.norm2, cfg.eps)
        g, u = (h @ self.w13.t()).chunk(2, dim=-1)
        return x + (F.silu(g) * u) @ self.w2.t()


class LlamaDecoder(nn.Module):
    """Compiled body: embedding -> blocks -> final norm (hidden states out)."""

    def __init__(self, cfg: LlamaConfig, dtype=torch.bfloat16, device=None, init_std=0.02,
                 fused: bool = True):
        super().__init__()
        self.cfg = cfg
        self.fused = fused
        kw = dict(dtype=dtype, device=device)
        self.embed = nn.Parameter(torch.empty(cfg.vocab, cfg.d_model, **kw))
        self.blocks = nn.ModuleList(LlamaBlock(cfg, dtype, device, fused)
                                    for _ in range(cfg.layers))
        self.norm = nn.Parameter(torch.ones(cfg.d_model, **kw))
        self.lm_head = nn.Parameter(torch.empty(cfg.vocab, cfg.d_model, **kw))
        inv = 1.0 / (cfg.rope_theta ** (torch.arange(0, cfg.head_dim, 2, dtype=torch.float32,
                                                         device=device) / cfg.head_dim))
        self.register_buffer("inv_freq", inv, persistent=False)
        with torch.no_grad():
            for p in self.parameters():
                if p.dim() == 2:
                    p.normal_(0.0, init_std)

    def forward(self, ids: torch.Tensor) -> torch.Tensor:
        b, s = ids.shape
        pos = positions(s, device=ids.device).float()  # auto_sp adds rank * s/P
        cos = sin = None
        if not self.fused:
            fr = pos[:, None] * self.inv_freq[None, :]
            cos, sin = fr.cos(), fr.sin()
        x = F.embedding(ids, self.embed)
        for blk in self.blocks:
            x = blk(x, cos, sin, pos)
        if self.fused:
            from . import ops
            return ops.rms_norm(x, self.norm, self.cfg.eps)
        return rmsnorm(x, self.norm, self.cfg.eps)


class ChunkedLMLoss(torch.autograd.Function):
    """Sum of token cross-entropies without materialising [tokens, vocab] fp32 logits and
    without recomputing them: each bf16 logits chunk (cuBLAS) is reduced by the fused CE
    kernel and turned into dlogits IN PLACE right away (softmax - onehot, for an upstream
    gradient of 1), from which the chunk's dhidden and dweight are produced in the same
    pass -- 3 vocab-sized GEMMs per chunk instead of 4 (forward logits + backward logits
    recompute + 2 gradient GEMMs).  The backward only scales the stored gradients by the
    upstream gradient."""

    @staticmethod
    def forward(ctx, hidden, weight, labels, chunk):
        from . import kernels
        n = hidden.shape[0]
        total = torch.zeros((), dtype=torch.float32, device=hidden.device)
        dh = torch.empty_like(hidden)
        dw = torch.zeros_like(weight)
        for i in range(0, n, chunk):
            h = hidden[i:i + chunk]
            logits = h @ weight.t()
            lse, loss = kernels.ce_fwd(logits, labels[i:i + chunk])
            total += loss.sum()
            dl = kernels.ce_bwd_(logits, labels[i:i + chunk], lse, 1.0)
            torch.matmul(dl, weight, out=dh[i:i + chunk])
            dw.addmm_(dl.t(), h)
        ctx.save_for_backward(dh, dw)
        return total

    @staticmethod
    def backward(ctx, g):
        dh, dw = ctx.saved_tensors
        g = g.to(dh.dtype)
        return dh * g, dw * g, None, None


def lm_loss(hidden: torch.Tensor, weight: torch.Tensor, labels: torch.Tensor,
            chunk: int = 4096) -> torch.Tensor:
    """SUM of the token cross-entropies of ``hidden @ weight.T`` against ``labels``.
    Labels outside [0, vocab) (e.g. -100 padding) are ignored: they add 0 to the loss and
    get an all-zero gradient row (torch's ignore_index, with reduction='sum')."""
    h = hidden.reshape(-1, hidden.shape[-1])
    return ChunkedLMLoss.apply(h, weight, labels.reshape(-1), chunk)


def attention_flops_causal(b: int, hq: int, s: int, d: int) -> float:
    """Algorithmic causal attention forward FLOPs (2 GEMMs over the lower triangle)."""
    return 4.0 * b * hq * d * s * (s + 1) / 2


def train_flops_per_step(cfg: LlamaConfig, b: int, s: int) -> float:
    """6 * params * tokens for the dense layers + attention fwd (1x) + bwd (2.5x)."""
    dense = 6.0 * (cfg.n_params() - cfg.vocab * cfg.d_model) * b * s
    return dense + 3.5 * cfg.layers * attention_flops_causal(b, cfg.hq, s, cfg.head_dim)
