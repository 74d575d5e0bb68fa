"""TEST-ONLY CPU lowering of the AutoSP custom ops (never imported by the product path).

The sm_100a kernels have no CPU implementation; multi-process CPU tests (gloo,
world_size 2) still need to run the auto_sp/sp_ac graphs end to end.  This module
registers CPU kernels for ``autosp::attention``, ``autosp::attention_backward`` and
``autosp::all_to_all``: a plain-math attention and an all-gather-based all-to-all with
the reference's semantics (``executor.py:132-142, 203-230``)."""

from __future__ import annotations

import math

import torch
import torch.distributed as tdist

_ENABLED = False


def _attn_math(q, k, v, scale, causal):
    hq, hkv = q.shape[1], k.shape[1]
    ke = k.repeat_interleave(hq // hkv, dim=1)
    ve = v.repeat_interleave(hq // hkv, dim=1)
    sc = (q @ ke.transpose(-1, -2)) * scale
    if causal:
        s = q.shape[2]
        sc = sc + torch.triu(torch.full((s, s), -1e9, dtype=sc.dtype), diagonal=1)
    return sc, ke, ve


def enable_cpu_lowering() -> None:
    global _ENABLED
    if _ENABLED:
        return
    from paper_2604_27089_b200 import dist as sp_dist
    from paper_2604_27089_b200 import ops  # noqa: F401  (defines the ops)

    @torch.library.register_kernel("autosp::attention", "cpu")
    def _attention_cpu(q, k, v, scale, causal):
        sc, ke, ve = _attn_math(q, k, v, scale, causal)
        lse = torch.logsumexp(sc, dim=-1)
        o = torch.softmax(sc, dim=-1) @ ve
        # same memory layout as the CUDA op (token-major, see ops.attention)
        return o.transpose(1, 2).contiguous().transpose(1, 2), lse.float()

    @torch.library.register_kernel("autosp::attention_backward", "cpu")
    def _attention_backward_cpu(do, q, k, v, o, lse, scale, causal):
        sc, ke, ve = _attn_math(q, k, v, scale, causal)
        p = torch.softmax(sc, dim=-1)
        dp = do @ ve.transpose(-1, -2)
        ds = p * (dp - (dp * p).sum(-1, keepdim=True)) * scale
        dq = ds @ ke
        g = q.shape[1] // k.shape[1]
        dk = (ds.transpose(-1, -2) @ q).unflatten(1, (k.shape[1], g)).sum(2)
        dv = (p.transpose(-1, -2) @ do).unflatten(1, (k.shape[1], g)).sum(2)
        return dq, dk, dv

    @torch.library.register_kernel("autosp::grad_out_reshard", "cpu")
    def _grad_out_reshard_cpu(d_otok, o_tok, group):
        acc = torch.promote_types(d_otok.dtype, torch.float32)
        delta_tok = (d_otok.to(acc) * o_tok.to(acc)).sum(-1, keepdim=True)
        (do,) = ops.all_to_all([d_otok], ops.SEQ_TO_HEAD_DIR, group)
        (delta,) = ops.all_to_all([delta_tok], ops.SEQ_TO_HEAD_DIR, group)
        return do, delta.squeeze(-1).contiguous()

    @torch.library.register_kernel("autosp::all_to_all", "cpu")
    def _all_to_all_cpu(xs, direction, group):
        st = sp_dist.lookup(group)
        P = st.world
        outs = []
        for x in xs:
            parts = [torch.empty_like(x.contiguous()) for _ in range(P)]
            if P > 1:
                tdist.all_gather(parts, x.contiguous(), group=st.group)
            else:
                parts = [x.contiguous()]
            shape, strides = ops._out_geometry(x, direction, P)
            if direction == ops.SEQ_TO_HEAD_DIR:  # parts [b, h, s/P, d] -> heads of my block
                hl = x.shape[1] // P
                full = torch.cat([p[:, st.rank * hl:(st.rank + 1) * hl] for p in parts], dim=2)
            else:  # parts [b, h/P, s, d] -> my tokens of every rank's heads
                sl = x.shape[2] // P
                full = torch.cat([p[:, :, st.rank * sl:(st.rank + 1) * sl] for p in parts], dim=1)
            out = torch.empty_strided(shape, strides, dtype=x.dtype)
            out.copy_(full)
            outs.append(out)
        return outs

    @torch.library.register_kernel("autosp::attention_a2a", "cpu")
    def _attention_a2a_cpu(q, k, v, scale, causal, group):
        o, lse = _attention_cpu(q, k, v, scale, causal)
        (ot,) = _all_to_all_cpu([o], ops.HEAD_TO_SEQ_DIR, group)
        return ot, lse

    @torch.library.register_kernel("autosp::attention_backward_delta", "cpu")
    def _attention_backward_delta_cpu(do, q, k, v, delta, lse, scale, causal):
        sc, ke, ve = _attn_math(q, k, v, scale, causal)
        p = torch.softmax(sc, dim=-1)
        dp = do @ ve.transpose(-1, -2)
        ds = p * (dp - delta.to(dp.dtype).unsqueeze(-1)) * scale
        dq = ds @ ke
        g = q.shape[1] // k.shape[1]
        dk = (ds.transpose(-1, -2) @ q).unflatten(1, (k.shape[1], g)).sum(2)
        dv = (p.transpose(-1, -2) @ do).unflatten(1, (k.shape[1], g)).sum(2)
        return dq, dk, dv

    _ENABLED = True


def loopback_states(P: int, nbytes: int, device="cuda", prefix: str = "loop"):
    """P virtual SP ranks on ONE GPU (test / single-GPU bench harness): every rank's
    receive region and flag block is a local allocation and each rank's pool maps all of
    them, so the real push kernels and epoch protocol run unchanged.  Returns the
    SPStates (group names f"{prefix}{r}") and the backing buffers (keep them alive)."""
    from paper_2604_27089_b200 import dist as sp_dist
    flags = torch.zeros((P, 1024), dtype=torch.int32, device=device)
    regions = [torch.empty(nbytes, dtype=torch.uint8, device=device) for _ in range(P)]
    peers = [(flags[j].data_ptr(), regions[j].data_ptr()) for j in range(P)]
    states = []
    for r in range(P):
        pool = sp_dist.SymmetricPool(nbytes, P, r, torch.device(device), peers=peers,
                                     reuse=False)
        st = sp_dist.SPState(world=P, rank=r, group=None, device=torch.device(device),
                             pool=pool, name=f"{prefix}{r}")
        sp_dist._REGISTRY[st.name] = st
        states.append(st)
    return states, (flags, regions)
