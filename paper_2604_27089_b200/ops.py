"""torch.library custom ops that the ``auto_sp`` pass lowers attention to.

    autosp::attention(q, k, v, scale, causal) -> (o, lse)          K3 (attn_fwd.cu)
    autosp::attention_backward(do, q, k, v, o, lse, ...) -> dq,dk,dv K4 (attn_bwd.cu)
    autosp::all_to_all(xs, direction, group) -> ys                 K1/K2 (a2a.cu)
    autosp::attention_a2a(q, k, v, scale, causal, group)           K3 + K2 fused
        -> (o_tokens, o_heads, lse)                                (attn_fwd.cu push epilogue)

All tensors use the SDPA logical layout ``[b, h, s, d]`` (head_dim contiguous, any
other strides).  ``all_to_all`` is the reference's AllToAll node
(``sp_pass.py:172-195``, ``executor.py:203-230``) over up to four tensors in ONE kernel
launch; its gradient is the inverse-direction all-to-all (``autodiff.py:252-262``).

The ops have CUDA kernels only.  There is no CPU kernel in the product: calling them on
CPU tensors raises.  (``tests/autosp_cpu_lowering.py``: ``enable_cpu_lowering()`` registers a test-only CPU/gloo
lowering used by the multi-process CPU tests.)
"""

from __future__ import annotations

import math

import torch

from . import dist as sp_dist
from . import _lib, kernels
from ._lib import HEAD_TO_SEQ, SEQ_TO_HEAD
from .errors import ValidationError

SEQ_TO_HEAD_DIR = SEQ_TO_HEAD
HEAD_TO_SEQ_DIR = HEAD_TO_SEQ
# The sm_100a attention computes in bf16 (fp32 accumulation); q/k/v of other dtypes are
# cast before the all-to-all (half the NVLink bytes) and the output cast back.
ATTN_DTYPE: torch.dtype | None = torch.bfloat16


# ----------------------------------------------------------------------------- attention
def _kernel_head_dim(d: int) -> int:
    """Head dims the sm_100a kernels implement are 32/64/128; smaller ones (the reference
    model's tiny configs use d = 4 / 8) run zero-padded to the next one: zero columns add
    nothing to q.k or p.v, so the result is unchanged (the scale stays 1/sqrt(d))."""
    for dp in kernels.SUPPORTED_HEAD_DIMS:
        if d <= dp:
            return dp
    raise ValidationError(f"head_dim {d} > {kernels.SUPPORTED_HEAD_DIMS[-1]} is not supported")


def _pad_d(t: torch.Tensor, dp: int) -> torch.Tensor:
    return torch.nn.functional.pad(t, (0, dp - t.shape[-1]))


@torch.library.custom_op("autosp::attention", mutates_args=(), device_types="cuda")
def attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, scale: float,
              causal: bool) -> tuple[torch.Tensor, torch.Tensor]:
    # O is written token-major ([b, s, h, d] memory, returned as the [b, h, s, d] view):
    # the caller's transpose(1, 2).reshape(b, s, h*d) before the O projection is then a
    # free view instead of a copy of the whole output
    b, h, s, d = q.shape
    o = torch.empty((b, s, h, d), dtype=q.dtype, device=q.device).transpose(1, 2)
    dp = _kernel_head_dim(d)
    if dp != d:
        op, lse = kernels.attn_fwd(_pad_d(q, dp), _pad_d(k, dp), _pad_d(v, dp), causal=causal,
                                   scale=scale)
        o.copy_(op[..., :d])
        return o, lse
    return kernels.attn_fwd(q, k, v, causal=causal, scale=scale, out=o)


@attention.register_fake
def _attention_fake(q, k, v, scale, causal):
    b, h, s, d = q.shape
    return (q.new_empty_strided((b, h, s, d), (s * h * d, d, h * d, 1)),
            q.new_empty((b, h, s), dtype=torch.float32))


@torch.library.custom_op("autosp::attention_backward", mutates_args=(), device_types="cuda")
def attention_backward(do: torch.Tensor, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor,
                       o: torch.Tensor, lse: torch.Tensor, scale: float,
                       causal: bool) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    if do.stride(-1) != 1:
        do = do.contiguous()
    d = q.shape[-1]
    dp = _kernel_head_dim(d)
    if dp != d:
        gs = kernels.attn_bwd(*(_pad_d(t, dp) for t in (q, k, v, o, do)), lse, causal=causal,
                              scale=scale)
        return tuple(g[..., :d].contiguous() for g in gs)
    return kernels.attn_bwd(q, k, v, o, do, lse, causal=causal, scale=scale)


@attention_backward.register_fake
def _attention_backward_fake(do, q, k, v, o, lse, scale, causal):
    return (q.new_empty(q.shape), k.new_empty(k.shape), v.new_empty(v.shape))


@torch.library.custom_op("autosp::attention_backward_delta", mutates_args=(), device_types="cuda")
def attention_backward_delta(do: torch.Tensor, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor,
                             delta: torch.Tensor, lse: torch.Tensor, scale: float,
                             causal: bool) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """attention_backward with delta = rowsum(dO * O) supplied (no O needed)."""
    if do.stride(-1) != 1:
        do = do.contiguous()
    d = q.shape[-1]
    dp = _kernel_head_dim(d)
    if dp != d:
        gs = kernels.attn_bwd(*(_pad_d(t, dp) for t in (q, k, v)), None, _pad_d(do, dp), lse,
                              causal=causal, scale=scale, delta=delta.float().contiguous())
        return tuple(g[..., :d].contiguous() for g in gs)
    return kernels.attn_bwd(q, k, v, None, do, lse, causal=causal, scale=scale,
                            delta=delta.float().contiguous())


@attention_backward_delta.register_fake
def _attention_backward_delta_fake(do, q, k, v, delta, lse, scale, causal):
    return (q.new_empty(q.shape), k.new_empty(k.shape), v.new_empty(v.shape))


def _attn_setup(ctx, inputs, output):
    q, k, v, scale, causal = inputs
    o, lse = output
    ctx.save_for_backward(q, k, v, o, lse)
    ctx.scale, ctx.causal = scale, causal


def _attn_bwd(ctx, do, dlse):
    q, k, v, o, lse = ctx.saved_tensors
    dq, dk, dv = attention_backward(do, q, k, v, o, lse, ctx.scale, ctx.causal)
    return dq, dk, dv, None, None


attention.register_autograd(_attn_bwd, setup_context=_attn_setup)


def _cast_in(*ts):
    if ATTN_DTYPE is None or ts[0].dtype == ATTN_DTYPE:
        return ts, None
    cast = {}
    for t in ts:  # keep aliasing (q = k = v in the reference model)
        if id(t) not in cast:
            cast[id(t)] = t.to(ATTN_DTYPE)
    return tuple(cast[id(t)] for t in ts), ts[0].dtype


def _sdpa(q, k, v, is_causal, scale):
    if not is_causal:
        raise ValidationError("auto_sp attention is causal (reference mask, executor.py:62-65)")
    scale = 1.0 / math.sqrt(q.shape[-1]) if scale is None else float(scale)
    return attention(q, k, v, scale, True)[0]


def sdpa(q, k, v, is_causal=True, scale=None):
    """Drop-in for F.scaled_dot_product_attention(q, k, v, is_causal=True[, enable_gqa])."""
    (q, k, v), dt = _cast_in(q, k, v)
    o = _sdpa(q, k, v, is_causal, scale)
    return o if dt is None else o.to(dt)


# ----------------------------------------------------------------------------- all-to-all
def _out_geometry(x: torch.Tensor, direction: int, P: int):
    """Logical output shape/strides for one [b, h, s, d] input."""
    b, h, s, d = x.shape
    if direction == SEQ_TO_HEAD_DIR:
        if h % P:
            raise ValidationError(f"heads {h} not divisible by world size {P}")
        hl, S = h // P, s * P
        shape = (b, hl, S, d)
        strides = (hl * S * d, S * d, d, 1)  # head-major: the attention operand layout
    else:
        if s % P:
            raise ValidationError(f"sequence {s} not divisible by world size {P}")
        H, sl = h * P, s // P
        shape = (b, H, sl, d)
        strides = (sl * H * d, d, H * d, 1)  # token-major: feeds the O projection directly
    return shape, strides


@torch.library.custom_op("autosp::all_to_all", mutates_args=(), device_types="cuda")
def all_to_all(xs: list[torch.Tensor], direction: int, group: str) -> list[torch.Tensor]:
    st = sp_dist.lookup(group)
    P = st.world
    if P == 1:
        return [x.clone() for x in xs]  # executor.py:208-209 (P == 1 -> copy)
    pool = st.pool
    descs, outs = [], []
    b, _, s, d = xs[0].shape
    xs = [x if x.stride(-1) == 1 else x.contiguous() for x in xs]
    geo = [_out_geometry(x, direction, P) for x in xs]
    # ONE slab per call (all destinations in the same segment, one peer-base array)
    slab = pool.alloc_many([math.prod(sh) * x.element_size() for x, (sh, _) in zip(xs, geo)])
    for x, (shape, strides), (off, base) in zip(xs, geo, slab.pieces):
        outs.append(base.view(x.dtype).as_strided(shape, strides))
        # kernel convention: logical [b, s, h, d] element strides of source and destination
        src_bshd = x.permute(0, 2, 1, 3)
        descs.append(kernels.a2a_tensor_desc(src_bshd, x.shape[1], off,
                                             (strides[0], strides[2], strides[1])))
    s_glob = s * P if direction == SEQ_TO_HEAD_DIR else s
    epoch = pool.next_epoch()
    chk = kernels.a2a_launch(direction, descs, b, s_glob, d, xs[0].element_size(), P, st.rank,
                             slab.regions, pool.flag_ptrs, epoch)
    kernels.a2a_wait(pool.flag_ptrs[st.rank], P, st.rank, epoch, chk)
    return outs


@all_to_all.register_fake
def _all_to_all_fake(xs, direction, group):
    P = sp_dist.lookup(group).world
    outs = []
    for x in xs:
        shape, strides = _out_geometry(x, direction, P)
        outs.append(x.new_empty_strided(shape, strides))
    return outs


def _a2a_setup(ctx, inputs, output):
    _, direction, group = inputs
    ctx.direction, ctx.group = direction, group


def _a2a_bwd(ctx, grads):
    inv = HEAD_TO_SEQ_DIR if ctx.direction == SEQ_TO_HEAD_DIR else SEQ_TO_HEAD_DIR
    return all_to_all(list(grads), inv, ctx.group), None, None


def _a2a_setup_shapes(ctx, inputs, output):
    _a2a_setup(ctx, inputs, output)


all_to_all.register_autograd(_a2a_bwd, setup_context=_a2a_setup)


# ----------------------------------------------------------------------------- fused K3 + K2
@torch.library.custom_op("autosp::attention_a2a", mutates_args=(), device_types="cuda")
def attention_a2a(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, scale: float, causal: bool,
                  group: str) -> tuple[torch.Tensor, torch.Tensor]:
    """Attention over the full sequence on the local heads whose epilogue pushes every
    output row to its token owner (the head->seq all-to-all, sp_pass.py:172-195, fused
    into the producing kernel).  Returns (o_tokens [b, H, s/P, d] token-major = the
    all-to-all output, lse [b, h/P, s]).  No head-major copy of O is kept: the backward
    forms delta = rowsum(dO * O) on the token owner (see _attn_a2a_bwd)."""
    st = sp_dist.lookup(group)
    P, pool = st.world, st.pool
    b, hl, S, d = q.shape
    lse = torch.empty((b, hl, S), dtype=torch.float32, device=q.device)
    shape, strides = _out_geometry(q, HEAD_TO_SEQ_DIR, P)  # (O has q's shape)
    slab = pool.alloc(math.prod(shape) * q.element_size())
    o_tok = slab.view.view(q.dtype).as_strided(shape, strides)
    epoch = pool.next_epoch()
    chk = kernels.attn_fwd_push(q, k, v, None, lse, scale, causal, P, st.rank, slab.offset,
                                (strides[0], strides[2], strides[1]), slab.regions,
                                pool.flag_ptrs, epoch)
    kernels.a2a_wait(pool.flag_ptrs[st.rank], P, st.rank, epoch, chk)
    return o_tok, lse


@attention_a2a.register_fake
def _attention_a2a_fake(q, k, v, scale, causal, group):
    P = sp_dist.lookup(group).world
    b, hl, S, d = q.shape
    shape, strides = _out_geometry(q, HEAD_TO_SEQ_DIR, P)
    return (q.new_empty_strided(shape, strides), q.new_empty((b, hl, S), dtype=torch.float32))


def _attn_a2a_setup(ctx, inputs, output):
    q, k, v, scale, causal, group = inputs
    o_tok, lse = output
    ctx.save_for_backward(q, k, v, o_tok, lse)
    ctx.scale, ctx.causal, ctx.group = scale, causal, group


@torch.library.custom_op("autosp::grad_out_reshard", mutates_args=(), device_types="cuda")
def grad_out_reshard(d_otok: torch.Tensor, o_tok: torch.Tensor,
                     group: str) -> tuple[torch.Tensor, torch.Tensor]:
    """The backward's first reshard (the inverse of the fused head->seq push of O,
    autodiff.py:252-262): dO seq->head, head-major [b, h/P, S, d], together with
    delta = rowsum(dO * O) [b, h/P, S] fp32 -- formed on the token owner, where the
    token-major O already is (kept for the O-projection weight gradient), in the SAME push
    kernel (autosp_a2a_grad_out: one launch instead of an fp32 elementwise product, a
    reduction and two reshards)."""
    st = sp_dist.lookup(group)
    P, pool = st.world, st.pool
    b, H, sl, d = d_otok.shape
    if P == 1 or d_otok.dtype != torch.bfloat16 or d not in kernels.SUPPORTED_HEAD_DIMS or \
            o_tok.dtype != torch.bfloat16:
        delta_tok = (d_otok.float() * o_tok.float()).sum(-1, keepdim=True)
        (do,) = all_to_all([d_otok], SEQ_TO_HEAD_DIR, group)
        (delta,) = all_to_all([delta_tok], SEQ_TO_HEAD_DIR, group)
        return do, delta.squeeze(-1).contiguous()
    if H % P:
        raise ValidationError(f"heads {H} not divisible by world size {P}")
    hl, S = H // P, sl * P
    slab = pool.alloc_many([b * hl * S * d * 2, b * hl * S * 4])
    (off0, p0), (off1, p1) = slab.pieces
    do = p0.view(torch.bfloat16).as_strided((b, hl, S, d), (hl * S * d, S * d, d, 1))
    delta = p1.view(torch.float32).view(b, hl, S)
    t0 = kernels.a2a_tensor_desc(d_otok.permute(0, 2, 1, 3), H, off0, (hl * S * d, d, S * d))
    t1 = kernels.a2a_tensor_desc(o_tok.permute(0, 2, 1, 3), H, off1, (hl * S, 1, S))
    epoch = pool.next_epoch()
    chk = kernels.a2a_grad_out(t0, t1, b, S, d, P, st.rank, slab.regions, pool.flag_ptrs, epoch)
    kernels.a2a_wait(pool.flag_ptrs[st.rank], P, st.rank, epoch, chk)
    return do, delta


@grad_out_reshard.register_fake
def _grad_out_reshard_fake(d_otok, o_tok, group):
    P = sp_dist.lookup(group).world
    b, H, sl, d = d_otok.shape
    hl, S = H // P, sl * P
    return (d_otok.new_empty_strided((b, hl, S, d), (hl * S * d, S * d, d, 1)),
            d_otok.new_empty((b, hl, S), dtype=torch.float32))


def ulysses_attention_grad(d_otok, o_tok, q, k, v, lse, scale, causal, group):
    """Backward of the fused attention + head->seq reshard: delta = rowsum(dO * O) is
    formed on the token owner from the token-major output (kept anyway for the
    O-projection weight gradient) and resharded with dO in one push (grad_out_reshard,
    the inverse all-to-all of the fused one, autodiff.py:252-262)."""
    do, delta = grad_out_reshard(d_otok, o_tok, group)
    return attention_backward_delta(do, q, k, v, delta, lse, scale, causal)


def _attn_a2a_bwd(ctx, d_otok, d_lse):
    q, k, v, o_tok, lse = ctx.saved_tensors
    dq, dk, dv = ulysses_attention_grad(d_otok, o_tok, q, k, v, lse, ctx.scale, ctx.causal,
                                        ctx.group)
    return dq, dk, dv, None, None, None


attention_a2a.register_autograd(_attn_a2a_bwd, setup_context=_attn_a2a_setup)

# ----------------------------------------------------------------------------- Ulysses block
# from the PACKED QKV projection output: RoPE + split + transpose folded into the reshard
@torch.library.custom_op("autosp::ulysses_qkv_attention", mutates_args=(), device_types="cuda")
def ulysses_qkv_attention(qkv: torch.Tensor, pos: torch.Tensor, theta: float, hq: int, hkv: int,
                          scale: float, group: str) -> tuple[torch.Tensor, torch.Tensor,
                                                             torch.Tensor, torch.Tensor,
                                                             torch.Tensor]:
    """The whole Ulysses attention block (sp_pass.py:172-195) fed by the packed projection
    output qkv [b, s/P, hq+2hkv, d] of this rank's tokens:
      K1 (a2a_rope): q/k rotated and v moved straight from the packed rows into the head
         owners' receive regions, head-major [b, h/P, s, d] -- the projection output is
         read once, no RoPE / split / transpose kernel;
      K3+K2: causal attention on the local heads, the epilogue pushing O to the token
         owners (token-major [b, H, s/P, d] = the O-projection input).
    Returns (o_tokens, q_heads, k_heads, v_heads, lse); with o_tokens these are what the
    backward needs (the a2a outputs sp_ac keeps; no head-major O)."""
    st = sp_dist.lookup(group)
    P, pool = st.world, st.pool
    b, sl, H3, d = qkv.shape
    S = sl * P
    if H3 != hq + 2 * hkv or hq % P or hkv % P:
        raise ValidationError(f"qkv heads {H3} != {hq}+2*{hkv} or not divisible by {P}")
    srcs = (qkv[:, :, :hq], qkv[:, :, hq:hq + hkv], qkv[:, :, hq + hkv:])
    outs, descs = [], []
    slab = pool.alloc_many([b * (x.shape[2] // P) * S * d * qkv.element_size() for x in srcs])
    for x, rot, (off, base) in zip(srcs, (True, True, False), slab.pieces):
        h = x.shape[2]
        shape = (b, h // P, S, d)
        strides = ((h // P) * S * d, S * d, d, 1)
        outs.append(base.view(qkv.dtype).as_strided(shape, strides))
        descs.append(kernels.a2a_tensor_desc(x, h, off, (strides[0], strides[2], strides[1]),
                                             rope=rot))
    epoch = pool.next_epoch()
    chk = kernels.a2a_launch(SEQ_TO_HEAD_DIR, descs, b, S, d, qkv.element_size(), P, st.rank,
                             slab.regions, pool.flag_ptrs, epoch,
                             pos=pos.to(torch.float32).contiguous(), theta=theta)
    kernels.a2a_wait(pool.flag_ptrs[st.rank], P, st.rank, epoch, chk)
    qh, kh, vh = outs
    o_tok, lse = attention_a2a(qh, kh, vh, scale, True, group)
    return o_tok, qh, kh, vh, lse


@ulysses_qkv_attention.register_fake
def _ulysses_qkv_attention_fake(qkv, pos, theta, hq, hkv, scale, group):
    P = sp_dist.lookup(group).world
    b, sl, H3, d = qkv.shape
    S = sl * P
    H = hq
    heads = lambda h: qkv.new_empty_strided((b, h // P, S, d), ((h // P) * S * d, S * d, d, 1))
    return (qkv.new_empty_strided((b, H, sl, d), (sl * H * d, d, H * d, 1)), heads(hq),
            heads(hkv), heads(hkv), qkv.new_empty((b, hq // P, S), dtype=torch.float32))


def _uqa_setup(ctx, inputs, output):
    qkv, pos, theta, hq, hkv, scale, group = inputs
    o_tok, qh, kh, vh, lse = output
    ctx.save_for_backward(pos, qh, kh, vh, o_tok, lse)
    ctx.theta, ctx.hq, ctx.hkv, ctx.scale, ctx.group = theta, hq, hkv, scale, group
    ctx.qkv_shape = tuple(qkv.shape)


FUSE_GRAD_A2A = True  # K4's epilogues push dq/dk/dv to the token owners (no separate K1)


def _uqa_bwd(ctx, d_otok, *unused):
    pos, qh, kh, vh, o_tok, lse = ctx.saved_tensors
    if FUSE_GRAD_A2A and qh.shape[-1] in kernels.SUPPORTED_HEAD_DIMS:
        do, delta = grad_out_reshard(d_otok, o_tok, ctx.group)
        dqkv = qkv_attention_grad(do, qh, kh, vh, delta, lse, pos, ctx.theta, ctx.scale,
                                  ctx.group)
        return dqkv, None, None, None, None, None, None
    dq, dk, dv = ulysses_attention_grad(d_otok, o_tok, qh, kh, vh, lse, ctx.scale, True,
                                        ctx.group)
    dqkv = qkv_grad_gather(dq, dk, dv, pos, ctx.theta, ctx.group)
    return dqkv, None, None, None, None, None, None


@torch.library.custom_op("autosp::qkv_attention_grad", mutates_args=(), device_types="cuda")
def qkv_attention_grad(do: torch.Tensor, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor,
                       delta: torch.Tensor, lse: torch.Tensor, pos: torch.Tensor, theta: float,
                       scale: float, group: str) -> torch.Tensor:
    """The attention backward (K4) with the head->seq all-to-all of its gradients fused
    into its epilogues (autodiff.py:252-262 + the attention recipes :156-214): dK/dV rows
    leave K4's epilogue and dQ rows its finalisation straight for the token owners'
    packed [b, s/P, hq+2hkv, d] QKV gradient (no local dq/dk/dv, no K1 launch); then the
    inverse RoPE of the q/k heads in place (one launch)."""
    st = sp_dist.lookup(group)
    P, pool = st.world, st.pool
    b, hql, S, d = q.shape
    hkvl = k.shape[1]
    hq, hkv, sl = hql * P, hkvl * P, S // P
    H3 = hq + 2 * hkv
    slab = pool.alloc(b * sl * H3 * d * q.element_size())
    dqkv = slab.view.view(q.dtype).as_strided((b, sl, H3, d), (sl * H3 * d, H3 * d, d, 1))
    epoch = pool.next_epoch()
    chk = kernels.attn_bwd_push(q, k, v, do, lse, delta.contiguous(), scale, True, P, st.rank,
                                slab.offset, (sl * H3 * d, H3 * d, d), slab.regions,
                                pool.flag_ptrs, epoch)
    kernels.a2a_wait(pool.flag_ptrs[st.rank], P, st.rank, epoch, chk)
    kernels.rope_segments([(dqkv[:, :, :hq], dqkv[:, :, :hq], True),
                           (dqkv[:, :, hq:hq + hkv], dqkv[:, :, hq:hq + hkv], True)],
                          pos, theta, inverse=True)
    return dqkv


@qkv_attention_grad.register_fake
def _qkv_attention_grad_fake(do, q, k, v, delta, lse, pos, theta, scale, group):
    P = sp_dist.lookup(group).world
    b, hql, S, d = q.shape
    H3 = (hql + 2 * k.shape[1]) * P
    return q.new_empty((b, S // P, H3, d))


ulysses_qkv_attention.register_autograd(_uqa_bwd, setup_context=_uqa_setup)


@torch.library.custom_op("autosp::qkv_grad_gather", mutates_args=(), device_types="cuda")
def qkv_grad_gather(dq: torch.Tensor, dk: torch.Tensor, dv: torch.Tensor, pos: torch.Tensor,
                    theta: float, group: str) -> torch.Tensor:
    """Backward of the RoPE-fused seq->head reshard: dq/dk/dv (head-sharded [b, h/P, s, d])
    pushed head->seq straight into ONE packed [b, s/P, hq+2hkv, d] gradient on each token
    owner, then the inverse rotation of its q/k heads in place (one segmented-RoPE launch)."""
    st = sp_dist.lookup(group)
    P, pool = st.world, st.pool
    b, hql, S, d = dq.shape
    hkvl = dk.shape[1]
    hq, hkv, sl = hql * P, hkvl * P, S // P
    H3 = hq + 2 * hkv
    es = dq.element_size()
    slab = pool.alloc(b * sl * H3 * d * es)
    off = slab.offset
    dqkv = slab.view.view(dq.dtype).as_strided((b, sl, H3, d), (sl * H3 * d, H3 * d, d, 1))
    descs = []
    for x, h0 in ((dq, 0), (dk, hq), (dv, hq + hkv)):
        if x.stride(-1) != 1:
            x = x.contiguous()
        descs.append(kernels.a2a_tensor_desc(x.permute(0, 2, 1, 3), x.shape[1], off + h0 * d * es,
                                             (sl * H3 * d, H3 * d, d)))
    epoch = pool.next_epoch()
    chk = kernels.a2a_launch(HEAD_TO_SEQ_DIR, descs, b, S, d, es, P, st.rank, slab.regions,
                             pool.flag_ptrs, epoch)
    kernels.a2a_wait(pool.flag_ptrs[st.rank], P, st.rank, epoch, chk)
    kernels.rope_segments([(dqkv[:, :, :hq], dqkv[:, :, :hq], True),
                           (dqkv[:, :, hq:hq + hkv], dqkv[:, :, hq:hq + hkv], True)],
                          pos, theta, inverse=True)
    return dqkv


@qkv_grad_gather.register_fake
def _qkv_grad_gather_fake(dq, dk, dv, pos, theta, group):
    P = sp_dist.lookup(group).world
    b, hql, S, d = dq.shape
    H3 = (hql + 2 * dk.shape[1]) * P
    return dq.new_empty((b, S // P, H3, d))


def ulysses_qkv_block(qkv, pos, theta: float, hq: int, hkv: int, group: str, scale=None):
    """What auto_sp substitutes for qkv_rope -> transpose -> SDPA at P > 1 (bf16)."""
    sc = 1.0 / math.sqrt(qkv.shape[-1]) if scale is None else float(scale)
    return ulysses_qkv_attention(qkv, pos, theta, hq, hkv, sc, group)[0]


def qkv_proj_fusable(h_shape, w_shape, hq: int, hkv: int) -> bool:
    """K0's tile constraints (autosp_qkv_gemm): 128-token tiles of every batch element,
    256-column output tiles, 64-deep K blocks."""
    b, sl, K = h_shape
    N = w_shape[0]
    d = N // (hq + 2 * hkv)
    return (sl % 128 == 0 and N % 256 == 0 and K % 64 == 0 and d in (32, 64, 128) and
            w_shape[1] == K and N == (hq + 2 * hkv) * d)


def ulysses_qkv_proj_block(h, w, pos, theta: float, hq: int, hkv: int, group: str, scale=None):
    """What auto_sp substitutes for h @ wqkv.t() -> qkv_rope -> transpose -> SDPA at P > 1
    when K0's tile constraints hold: the projection GEMM pushes RoPE'd head-major q/k/v
    rows to their owners from its epilogue."""
    d = w.shape[0] // (hq + 2 * hkv)
    sc = 1.0 / math.sqrt(d) if scale is None else float(scale)
    return ulysses_qkv_proj_attention(h, w, pos, theta, hq, hkv, sc, group)[0]


@torch.library.custom_op("autosp::ulysses_qkv_proj_attention", mutates_args=(),
                         device_types="cuda")
def ulysses_qkv_proj_attention(h: torch.Tensor, w: torch.Tensor, pos: torch.Tensor, theta: float,
                               hq: int, hkv: int, scale: float,
                               group: str) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor,
                                                    torch.Tensor, torch.Tensor]:
    """The Ulysses attention block from the projection INPUT h [b, s/P, K] (sp_pass.py:
    172-195 with the projection Linear of transformer.py:66-72 in front):
      K0 (autosp_qkv_gemm): Y = h W^T on the tensor cores, each (token, head) row of the
         epilogue RoPE-rotated (q/k) and pushed head-major [b, h/P, s, d] into its
         owner's receive region -- the reshard overlaps the GEMM, and the packed
         projection output is never written to HBM;
      K3+K2: causal attention on the local heads, O pushed back to the token owners.
    Returns (o_tokens, q_heads, k_heads, v_heads, lse) like ulysses_qkv_attention."""
    st = sp_dist.lookup(group)
    P, pool = st.world, st.pool
    b, sl, K = h.shape
    N = w.shape[0]
    d = N // (hq + 2 * hkv)
    S = sl * P
    if not qkv_proj_fusable(tuple(h.shape), tuple(w.shape), hq, hkv) or hq % P or hkv % P:
        raise ValidationError(f"ulysses_qkv_proj_attention: shapes {tuple(h.shape)} x "
                              f"{tuple(w.shape)} ({hq}/{hkv} heads, P={P}) not supported by K0")
    x2 = h.reshape(b * sl, K)
    if x2.stride(1) != 1:
        x2 = x2.contiguous()
    slab = pool.alloc_many([b * (x // P) * S * d * h.element_size() for x in (hq, hkv, hkv)])
    outs, dst3 = [], []
    for x, (off, base) in zip((hq, hkv, hkv), slab.pieces):
        shape = (b, x // P, S, d)
        strides = ((x // P) * S * d, S * d, d, 1)
        outs.append(base.view(h.dtype).as_strided(shape, strides))
        dst3.append(_lib.A2ATensor(None, 0, 0, 0, off, strides[0], strides[2], strides[1], x, 0))
    epoch = pool.next_epoch()
    chk = kernels.qkv_gemm(x2, w, hq, hkv, sl, pos=pos.to(torch.float32).contiguous(),
                           theta=theta, dst3=dst3, world=P, rank=st.rank,
                           peer_base=slab.regions, peer_flags=pool.flag_ptrs, epoch=epoch)
    kernels.a2a_wait(pool.flag_ptrs[st.rank], P, st.rank, epoch, chk)
    qh, kh, vh = outs
    o_tok, lse = attention_a2a(qh, kh, vh, scale, True, group)
    return o_tok, qh, kh, vh, lse


@ulysses_qkv_proj_attention.register_fake
def _uqpa_fake(h, w, pos, theta, hq, hkv, scale, group):
    P = sp_dist.lookup(group).world
    b, sl, _ = h.shape
    d = w.shape[0] // (hq + 2 * hkv)
    S = sl * P
    heads = lambda x: h.new_empty_strided((b, x // P, S, d), ((x // P) * S * d, S * d, d, 1))
    return (h.new_empty_strided((b, hq, sl, d), (sl * hq * d, d, hq * d, 1)), heads(hq),
            heads(hkv), heads(hkv), h.new_empty((b, hq // P, S), dtype=torch.float32))


def _uqpa_setup(ctx, inputs, output):
    h, w, pos, theta, hq, hkv, scale, group = inputs
    o_tok, qh, kh, vh, lse = output
    ctx.save_for_backward(h, w, pos, qh, kh, vh, o_tok, lse)
    ctx.theta, ctx.hq, ctx.hkv, ctx.scale, ctx.group = theta, hq, hkv, scale, group


def _uqpa_bwd(ctx, d_otok, *unused):
    """dqkv from K4 with its gradient push (qkv_attention_grad), then the projection's
    two gradient GEMMs (cuBLAS): dh = dqkv W, dW = dqkv^T h."""
    h, w, pos, qh, kh, vh, o_tok, lse = ctx.saved_tensors
    do, delta = grad_out_reshard(d_otok, o_tok, ctx.group)
    dqkv = qkv_attention_grad(do, qh, kh, vh, delta, lse, pos, ctx.theta, ctx.scale, ctx.group)
    b, sl, K = h.shape
    g2 = dqkv.reshape(b * sl, w.shape[0])
    dh = (g2 @ w).view(b, sl, K)
    dw = g2.t() @ h.reshape(b * sl, K)
    return dh, dw, None, None, None, None, None, None


ulysses_qkv_proj_attention.register_autograd(_uqpa_bwd, setup_context=_uqpa_setup)


FUSE_OUTPUT_A2A = True  # attention epilogue pushes O (K3 + K2 in one kernel)


def ulysses_attention(q, k, v, group: str, is_causal=True, scale=None):
    """The Ulysses attention block the auto_sp pass substitutes for SDPA
    (sp_pass.py:172-195): a2a seq->head of (q, k, v) in one launch, causal attention over
    the full sequence on the local heads, a2a head->seq of the output."""
    (q, k, v), dt = _cast_in(q, k, v)
    if k is v:  # reference model: q = k = v -> move the tensor once (transformer.py:3-6)
        kk = [q] if q is k else [q, k]
        moved = all_to_all(kk, SEQ_TO_HEAD_DIR, group)
        qh, kh = moved[0], moved[-1]
        vh = kh
    else:
        qh, kh, vh = all_to_all([q, k, v], SEQ_TO_HEAD_DIR, group)
    if FUSE_OUTPUT_A2A and qh.shape[-1] in kernels.SUPPORTED_HEAD_DIMS:
        if not is_causal:
            raise ValidationError("auto_sp attention is causal (reference mask, executor.py:62-65)")
        sc = 1.0 / math.sqrt(qh.shape[-1]) if scale is None else float(scale)
        o = attention_a2a(qh, kh, vh, sc, True, group)[0]
    else:
        oh = _sdpa(qh, kh, vh, is_causal, scale)
        (o,) = all_to_all([oh], HEAD_TO_SEQ_DIR, group)
    return o if dt is None else o.to(dt)


# ----------------------------------------------------------------------------- fused layer ops
# HBM-bound kernels for the layer around the Ulysses path (csrc/fused.cu); recomputable
# by sp_ac (never guarded).
@torch.library.custom_op("autosp::swiglu", mutates_args=(), device_types="cuda")
def swiglu(gu: torch.Tensor) -> torch.Tensor:
    return kernels.swiglu_fwd(gu)


@swiglu.register_fake
def _swiglu_fake(gu):
    return gu.new_empty((*gu.shape[:-1], gu.shape[-1] // 2))


@torch.library.custom_op("autosp::swiglu_backward", mutates_args=(), device_types="cuda")
def swiglu_backward(gu: torch.Tensor, dout: torch.Tensor) -> torch.Tensor:
    return kernels.swiglu_bwd(gu, dout)


@swiglu_backward.register_fake
def _swiglu_backward_fake(gu, dout):
    return gu.new_empty(gu.shape)


def _swiglu_setup(ctx, inputs, output):
    ctx.save_for_backward(inputs[0])


def _swiglu_bwd(ctx, dout):
    (gu,) = ctx.saved_tensors
    return swiglu_backward(gu, dout)


swiglu.register_autograd(_swiglu_bwd, setup_context=_swiglu_setup)


@torch.library.custom_op("autosp::rope", mutates_args=(), device_types="cuda")
def rope(x: torch.Tensor, pos: torch.Tensor, theta: float, inverse: bool) -> torch.Tensor:
    return kernels.rope(x, pos, theta, inverse)


@rope.register_fake
def _rope_fake(x, pos, theta, inverse):
    return x.new_empty(x.shape)


def _rope_setup(ctx, inputs, output):
    x, pos, theta, inverse = inputs
    ctx.save_for_backward(pos)
    ctx.theta, ctx.inverse = theta, inverse


def _rope_bwd(ctx, dy):
    (pos,) = ctx.saved_tensors
    if dy.stride(-1) != 1:
        dy = dy.contiguous()
    return rope(dy, pos, ctx.theta, not ctx.inverse), None, None, None


rope.register_autograd(_rope_bwd, setup_context=_rope_setup)


# QKV split + RoPE as one op: forward = one launch producing q, k (rotated) and v from the
# packed projection output; backward = one launch assembling the packed QKV gradient
# (replaces 2 rope launches + 3 zero-filled slice_backward buffers + 2 adds).
@torch.library.custom_op("autosp::qkv_rope", mutates_args=(), device_types="cuda")
def qkv_rope(qkv: torch.Tensor, pos: torch.Tensor, theta: float, hq: int,
             hkv: int) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    b, s, _, d = qkv.shape
    q = torch.empty((b, s, hq, d), dtype=qkv.dtype, device=qkv.device)
    k = torch.empty((b, s, hkv, d), dtype=qkv.dtype, device=qkv.device)
    v = torch.empty((b, s, hkv, d), dtype=qkv.dtype, device=qkv.device)
    kernels.rope_segments([(qkv[:, :, :hq], q, True), (qkv[:, :, hq:hq + hkv], k, True),
                           (qkv[:, :, hq + hkv:], v, False)], pos, theta, False)
    return q, k, v


@qkv_rope.register_fake
def _qkv_rope_fake(qkv, pos, theta, hq, hkv):
    b, s, _, d = qkv.shape
    return (qkv.new_empty((b, s, hq, d)), qkv.new_empty((b, s, hkv, d)),
            qkv.new_empty((b, s, hkv, d)))


@torch.library.custom_op("autosp::qkv_rope_backward", mutates_args=(), device_types="cuda")
def qkv_rope_backward(dq: torch.Tensor, dk: torch.Tensor, dv: torch.Tensor, pos: torch.Tensor,
                      theta: float) -> torch.Tensor:
    b, s, hq, d = dq.shape
    hkv = dk.shape[2]
    dqkv = torch.empty((b, s, hq + 2 * hkv, d), dtype=dq.dtype, device=dq.device)
    kernels.rope_segments([(dq, dqkv[:, :, :hq], True), (dk, dqkv[:, :, hq:hq + hkv], True),
                           (dv, dqkv[:, :, hq + hkv:], False)], pos, theta, True)
    return dqkv


@qkv_rope_backward.register_fake
def _qkv_rope_backward_fake(dq, dk, dv, pos, theta):
    b, s, hq, d = dq.shape
    return dq.new_empty((b, s, hq + 2 * dk.shape[2], d))


def _qkv_rope_setup(ctx, inputs, output):
    _, pos, theta, _, _ = inputs
    ctx.save_for_backward(pos)
    ctx.theta = theta


def _qkv_rope_bwd(ctx, dq, dk, dv):
    (pos,) = ctx.saved_tensors
    fix = lambda t: t if t.stride(-1) == 1 else t.contiguous()
    return qkv_rope_backward(fix(dq), fix(dk), fix(dv), pos, ctx.theta), None, None, None, None


qkv_rope.register_autograd(_qkv_rope_bwd, setup_context=_qkv_rope_setup)


# RMSNorm with a one-pass backward (dx and the weight gradient from one read of dy, x)
@torch.library.custom_op("autosp::rms_norm", mutates_args=(), device_types="cuda")
def rms_norm_op(x: torch.Tensor, w: torch.Tensor, eps: float) -> tuple[torch.Tensor, torch.Tensor]:
    return kernels.rms_norm_fwd(x, w, eps)


@rms_norm_op.register_fake
def _rms_norm_fake(x, w, eps):
    return x.new_empty(x.shape), x.new_empty(x.shape[:-1], dtype=torch.float32)


@torch.library.custom_op("autosp::rms_norm_backward", mutates_args=(), device_types="cuda")
def rms_norm_backward(dy: torch.Tensor, x: torch.Tensor, w: torch.Tensor,
                      rstd: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    return kernels.rms_norm_bwd(dy, x, w, rstd)


@rms_norm_backward.register_fake
def _rms_norm_backward_fake(dy, x, w, rstd):
    return x.new_empty(x.shape), w.new_empty(w.shape)


def _rms_setup(ctx, inputs, output):
    x, w, _ = inputs
    ctx.save_for_backward(x, w, output[1])


def _rms_bwd(ctx, dy, drstd):
    x, w, rstd = ctx.saved_tensors
    dx, dw = rms_norm_backward(dy, x, w, rstd)
    return dx, dw, None


rms_norm_op.register_autograd(_rms_bwd, setup_context=_rms_setup)


RMS_NORM_MAX_D = 4096  # measured (profiles/norm_bench_r01e.txt): fwd 1.2x / 1.0x, bwd 2.4x / 1.2x torch at d = 2048 / 4096


def rms_norm(x: torch.Tensor, w: torch.Tensor, eps: float) -> torch.Tensor:
    """Drop-in for F.rms_norm(x, (d,), w, eps) on CUDA bf16 (reference executor.py:43-45):
    the autosp kernels up to d = 2048 (tools/norm_bench.py), torch's fused RMSNorm above
    (it is not part of the Ulysses path; sp_ac recognises both)."""
    if x.shape[-1] > RMS_NORM_MAX_D:
        return torch.nn.functional.rms_norm(x, (x.shape[-1],), w, eps)
    return rms_norm_op(x, w, eps)[0]
