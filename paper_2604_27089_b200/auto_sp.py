"""``auto_sp`` — the Ulysses sequence-parallel rewrite on the Dynamo (Torch-IR) graph.

Reference: ``transform_sp`` (``sp_pass.py:133-220``).  Differences that follow from
running inside ``torch.compile`` instead of on a global desk-scale IR:

* the traced graph already sees each rank's sequence shard (the user feeds
  ``batch[:, sp_slice]``, paper Listing 1; reference ``shard_inputs``
  ``executor.py:324-341``), so RESIZE_BUFS need no rewrite — every shape outside
  attention is already ``s/P``;
* ATTN_OPS: every ``scaled_dot_product_attention`` call becomes
  a2a(seq->head) of (q, k, v) in one launch -> causal sm_100a attention over the full
  sequence on ``h/P`` heads -> a2a(head->seq)  (``sp_pass.py:172-195``);
* INDEX_OPS: position indices (``autosp.positions`` or integer ``torch.arange`` of the
  local sequence length) gain the rank offset ``rank * s/P`` (``sp_pass.py:160-163``,
  ``executor.py:68-70``); the causal mask stays implicit and full-sequence inside the
  kernel (``sp_pass.py:164-166``);
* errors mirror the reference: indivisible heads -> ValidationError
  (``sp_pass.py:145-148``), pass applied twice -> ValidationError (``sp_pass.py:134-135``).

At P = 1 the collectives are omitted (``sp_pass.py:138-144``) but attention is still
lowered to the sm_100a kernel.
"""

from __future__ import annotations

import operator
import warnings
from dataclasses import dataclass, field
from enum import Enum

import torch
import torch.fx as fx
import torch.nn.functional as F

from . import ops
from .dist import SPState
from .errors import ValidationError


class RewriteReason(str, Enum):  # sp_pass.py:34-37
    RESIZED_BUFFER = "ResizedBuffer"
    RECOMPUTED_INDEX = "RecomputedIndex"
    INSERTED_COLLECTIVE = "InsertedCollective"


ATTN_OPS = (torch._C._nn.scaled_dot_product_attention, F.scaled_dot_product_attention)


@torch.library.custom_op("autosp::positions", mutates_args=())
def _positions(n: int, device: torch.device) -> torch.Tensor:
    return torch.arange(n, device=device)


@_positions.register_fake
def _positions_fake(n, device):
    return torch.empty(n, dtype=torch.int64, device=device)


def positions(n: int, device=None) -> torch.Tensor:
    """Explicit position-index op (reference OpKind.POSITION_INDEX,
    ``executor.py:68-70``): the positions of the n tokens of THIS rank's shard.  auto_sp
    offsets it by rank * n.  An opaque graph node (not inlined into an arange), so it is
    found in any Dynamo subgraph, including one with no attention after a graph break.
    Equal to torch.arange(n) when run without the pass."""
    dev = torch.device(device) if device is not None else torch.get_default_device()
    return torch.ops.autosp.positions(n, dev)


_POSITIONS = (torch.ops.autosp.positions.default, torch.ops.autosp.positions)
INDEX_OPS = (*_POSITIONS, torch.arange)
_LOWERED = (ops.ulysses_attention, ops.sdpa, ops.ulysses_qkv_block)
FUSE_QKV_ROPE = True  # fold autosp::qkv_rope (RoPE + split + transpose) into the reshard
FUSE_QKV_PROJ = True  # and the projection GEMM in front of it (K0 pushes from its epilogue)


def _transposed_item(node, idx):
    """node == <x>.transpose(1, 2) with x == getitem(R, idx); returns R or None."""
    if not isinstance(node, fx.Node) or len(node.users) != 1:
        return None
    is_t = (node.op == "call_method" and node.target == "transpose") or \
        (node.op == "call_function" and node.target is torch.transpose)
    if not is_t or tuple(node.args[1:3]) not in ((1, 2), (2, 1)):
        return None
    it = node.args[0]
    if not (isinstance(it, fx.Node) and it.op == "call_function" and
            it.target is operator.getitem and it.args[1] == idx and len(it.users) == 1):
        return None
    return it.args[0]


def _match_qkv_rope(q, k, v):
    """q, k, v = transpose(getitem(autosp::qkv_rope(qkv, pos, theta, hq, hkv), i), 1, 2)
    for i = 0, 1, 2 of ONE qkv_rope node with no other users, bf16, d in {32, 64, 128}."""
    rs = [_transposed_item(x, i) for i, x in enumerate((q, k, v))]
    r = rs[0]
    if r is None or any(x is not r for x in rs):
        return None
    if not (r.op == "call_function" and r.target is torch.ops.autosp.qkv_rope.default and
            len(r.users) == 3):
        return None
    qkv = _val(r.args[0])
    if qkv is None or qkv.dtype != torch.bfloat16 or qkv.shape[-1] not in (32, 64, 128):
        return None
    return r


def _match_qkv_proj(rq):
    """qkv = view(matmul(h, t(w)), b, s, H3, d) feeding the matched qkv_rope, every link
    used once, within K0's tile constraints -> (view, matmul, t, h, w) else None."""
    qkv = rq.args[0]
    if not (isinstance(qkv, fx.Node) and qkv.op == "call_method" and
            qkv.target in ("view", "reshape") and len(qkv.users) == 1):
        return None
    mm = qkv.args[0]
    if not (isinstance(mm, fx.Node) and mm.op == "call_function" and
            mm.target in (operator.matmul, torch.matmul) and len(mm.users) == 1):
        return None
    h, tt = mm.args[:2]
    if not (isinstance(tt, fx.Node) and tt.op == "call_method" and tt.target == "t" and
            len(tt.users) == 1):
        return None
    w = tt.args[0]
    hv, wv = _val(h), _val(w)
    if hv is None or wv is None or hv.dim() != 3 or wv.dim() != 2 or \
            hv.dtype != torch.bfloat16 or wv.dtype != torch.bfloat16:
        return None
    if not ops.qkv_proj_fusable(tuple(hv.shape), tuple(wv.shape), rq.args[3], rq.args[4]):
        return None
    return qkv, mm, tt, h, w


@dataclass
class SPDims:  # reference infer_dims (sp_pass.py:102-123), on the local shard
    b: int
    s_local: int
    h: int
    d: int
    layers: int


@dataclass
class SPGraphInfo:
    world_size: int
    dims: SPDims | None  # None: a Dynamo subgraph without attention (graph break)
    provenance: dict[str, RewriteReason] = field(default_factory=dict)
    fused_qkv_proj: int = 0  # attention blocks whose projection GEMM pushes (K0)


def _val(n):
    v = n.meta.get("example_value", n.meta.get("val")) if isinstance(n, fx.Node) else n
    return v


def infer_dims(gm: fx.GraphModule, example_inputs) -> SPDims:
    attn = [n for n in gm.graph.nodes if n.op == "call_function" and n.target in ATTN_OPS]
    if not attn:
        raise ValidationError("graph has no attention node")
    qv = _val(attn[0].args[0])
    if qv is None or qv.dim() != 4:
        raise ValidationError("cannot read [b, h, s, d] from the first attention's query")
    b, h, s, d = qv.shape
    return SPDims(b=int(b), s_local=int(s), h=int(h), d=int(d), layers=len(attn))


def _token_input_len(gm: fx.GraphModule) -> int | None:
    """Local sequence length from the graph's single rank-2 integer input (the token ids;
    reference infer_dims reads b, s from "the single rank-2 input", sp_pass.py:102-123)."""
    cands = []
    for n in gm.graph.nodes:
        if n.op != "placeholder":
            continue
        v = _val(n)
        if isinstance(v, torch.Tensor) and v.dim() == 2 and not v.dtype.is_floating_point \
                and v.dtype != torch.bool:
            cands.append(int(v.shape[1]))
    return cands[0] if len(set(cands)) == 1 else None


def _is_int_arange_of(node: fx.Node, length: int) -> tuple[bool, int, int, int]:
    args = list(node.args)
    if not all(isinstance(a, int) for a in args):
        return False, 0, 0, 0
    dt = node.kwargs.get("dtype")
    if dt is not None and dt.is_floating_point:
        return False, 0, 0, 0
    if len(args) == 1:
        start, end, step = 0, args[0], 1
    elif len(args) == 2:
        start, end, step = args[0], args[1], 1
    elif len(args) == 3:
        start, end, step = args
    else:
        return False, 0, 0, 0
    n = max(0, (end - start + step - 1) // step) if step > 0 else 0
    return n == length and step == 1, start, end, step


def auto_sp(gm: fx.GraphModule, example_inputs, st: SPState) -> tuple[fx.GraphModule, SPGraphInfo]:
    g = gm.graph
    if any(n.op == "call_function" and n.target in _LOWERED for n in g.nodes):
        raise ValidationError("graph already lowered by auto_sp (pass already applied)")
    has_attn = any(n.op == "call_function" and n.target in ATTN_OPS for n in g.nodes)
    # a Dynamo subgraph without attention (the model graph-breaks, e.g. between the
    # embedding / positions and the first layer) is still rewritten: its position indices
    # need the rank offset.  positions(n) always denotes the local shard; a bare
    # torch.arange is matched against the local length read from the token-id input.
    dims = infer_dims(gm, example_inputs) if has_attn else None
    s_local = dims.s_local if dims is not None else _token_input_len(gm)
    P = st.world
    info = SPGraphInfo(world_size=P, dims=dims)
    for n in list(g.nodes):
        if n.op != "call_function":
            continue
        if n.target in ATTN_OPS:
            q, k, v = n.args[:3]
            kw = dict(n.kwargs)
            extra = list(n.args[3:])
            mask = kw.get("attn_mask", extra[0] if len(extra) > 0 else None)
            dropout = kw.get("dropout_p", extra[1] if len(extra) > 1 else 0.0)
            causal = kw.get("is_causal", extra[2] if len(extra) > 2 else False)
            scale = kw.get("scale", None)
            if mask is not None or not causal:
                raise ValidationError("auto_sp lowers causal attention only (mask must be implicit, "
                                      "reference executor.py:62-65)")
            if dropout:
                raise ValidationError("attention dropout is not supported")
            hq, hkv = _val(q).shape[1], _val(k).shape[1]
            if hq % P or hkv % P:
                raise ValidationError(f"head count {hq}/{hkv} not divisible by world size {P}")
            rq = _match_qkv_rope(q, k, v) if (P > 1 and FUSE_QKV_ROPE) else None
            proj = _match_qkv_proj(rq) if (rq is not None and FUSE_QKV_PROJ) else None
            with g.inserting_before(n):
                if proj is not None:
                    _, pos, theta, nq, nkv = rq.args[:5]
                    new = g.call_function(ops.ulysses_qkv_proj_block,
                                          (proj[3], proj[4], pos, theta, nq, nkv),
                                          {"group": st.name, "scale": scale})
                    info.provenance[new.name] = RewriteReason.INSERTED_COLLECTIVE
                    info.fused_qkv_proj += 1
                elif rq is not None:
                    qkv, pos, theta, nq, nkv = rq.args[:5]
                    new = g.call_function(ops.ulysses_qkv_block, (qkv, pos, theta, nq, nkv),
                                          {"group": st.name, "scale": scale})
                    info.provenance[new.name] = RewriteReason.INSERTED_COLLECTIVE
                elif P > 1:
                    new = g.call_function(ops.ulysses_attention, (q, k, v),
                                          {"group": st.name, "is_causal": True, "scale": scale})
                    info.provenance[new.name] = RewriteReason.INSERTED_COLLECTIVE
                else:
                    new = g.call_function(ops.sdpa, (q, k, v), {"is_causal": True, "scale": scale})
                    info.provenance[new.name] = RewriteReason.RESIZED_BUFFER
            new.meta.update(n.meta)
            n.replace_all_uses_with(new)
            g.erase_node(n)
            if rq is not None:  # the transposes, getitems and qkv_rope are now dead
                for x in (q, k, v):
                    it = x.args[0]
                    g.erase_node(x)
                    g.erase_node(it)
                g.erase_node(rq)
            if proj is not None:  # and the projection feeding it (view, matmul, t)
                for x in proj[:3]:
                    g.erase_node(x)
        elif n.target in INDEX_OPS and P > 1:
            if n.target in _POSITIONS:
                length = n.args[0]
                ok, start, end = isinstance(length, int), 0, length
                if not ok:
                    raise ValidationError("autosp.positions needs a static length")
                local = length
            else:
                if s_local is None:
                    if n.kwargs.get("dtype") is None or not n.kwargs["dtype"].is_floating_point:
                        warnings.warn("auto_sp: torch.arange in a subgraph with no attention and "
                                      "no token-id input is left unshifted; use "
                                      "autosp.positions(n) for position indices")
                    continue
                ok, start, end, _ = _is_int_arange_of(n, s_local)
                local = s_local
            if not ok or (end - start) != local:
                continue
            off = st.rank * local
            kwargs = {k: v for k, v in n.kwargs.items() if k in ("device", "dtype")}
            if n.target in _POSITIONS:
                kwargs = {"device": n.args[1] if len(n.args) > 1 else n.kwargs["device"]}
            with g.inserting_before(n):
                new = g.call_function(torch.arange, (start + off, end + off), kwargs)
            new.meta.update(n.meta)
            n.replace_all_uses_with(new)
            g.erase_node(n)
            info.provenance[new.name] = RewriteReason.RECOMPUTED_INDEX
    g.lint()
    gm.recompile()
    return gm, info
