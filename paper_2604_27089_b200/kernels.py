"""Torch-facing launchers of the sm_100a kernels in libautosp.so.

Tensors are passed as raw device pointers + strides through the C ABI (the library
never sees torch types).  All launches go on torch's current CUDA stream.  Nothing
here falls back to a PyTorch implementation: a missing library or a non-CUDA tensor
is an error."""

from __future__ import annotations

import ctypes as C
import math

import torch

from . import _lib
from .errors import ValidationError

SUPPORTED_HEAD_DIMS = (32, 64, 128)


class LaunchLog:
    """Counts the kernels this module launches and (optionally) times the attention
    calls with CUDA events on the launching stream (used by bench.py for the live
    roofline: algorithmic FLOPs per launch / measured launch duration)."""

    def __init__(self):
        self.enabled = False
        self.timing = False
        self.launches = 0
        self.events: dict[str, list] = {}
        self.flops: dict[str, float] = {}
        self.bytes: dict[str, float] = {}

    def reset(self, timing: bool = False):
        self.enabled, self.timing = True, timing
        self.launches = 0
        self.events, self.flops, self.bytes = {}, {}, {}

    def begin(self, name: str):
        if not (self.enabled and self.timing):
            return None
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        return e

    def end(self, name: str, start, n_kernels: int, flops: float = 0.0, nbytes: float = 0.0):
        if self.enabled:
            self.launches += n_kernels
        if start is not None:
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            self.events.setdefault(name, []).append((start, e))
            self.flops[name] = self.flops.get(name, 0.0) + flops
            self.bytes[name] = self.bytes.get(name, 0.0) + nbytes

    def summary(self) -> dict:
        out = {}
        for name, pairs in self.events.items():
            ms = sum(a.elapsed_time(b) for a, b in pairs)
            out[name] = {"calls": len(pairs), "ms": ms, "flops": self.flops.get(name, 0.0),
                         "bytes": self.bytes.get(name, 0.0)}
        return out


LOG = LaunchLog()


def causal_attn_flops(b: int, hq: int, s: int, d: int, causal: bool = True) -> float:
    """Algorithmic forward FLOPs: 2 GEMMs (QK^T, PV) over the unmasked (lower) triangle."""
    pairs = s * (s + 1) / 2 if causal else float(s) * s
    return 4.0 * b * hq * d * pairs


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _attn_tensor(t: torch.Tensor, name: str) -> _lib.AttnTensor:
    """[b, h, s, d] view, d contiguous."""
    if not t.is_cuda or t.dtype != torch.bfloat16:
        raise ValidationError(f"{name}: expected a CUDA bf16 tensor, got {t.device}/{t.dtype}")
    if t.dim() != 4 or t.stride(3) != 1:
        raise ValidationError(f"{name}: expected [b, h, s, d] with contiguous head_dim")
    sb, sh, ss, _ = t.stride()
    return _lib.AttnTensor(t.data_ptr(), sb, sh, ss)


def attn_fwd(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, causal: bool = True,
             scale: float | None = None, out: torch.Tensor | None = None):
    """Causal flash attention forward.  q [b, hq, s, d], k/v [b, hkv, s, d] (bf16 views).
    Returns (o [b, hq, s, d] bf16, lse [b, hq, s] fp32)."""
    lib = _lib.load()
    b, hq, s, d = q.shape
    hkv = k.shape[1]
    if k.shape != (b, hkv, s, d) or v.shape != k.shape:
        raise ValidationError(f"attn_fwd: q {tuple(q.shape)} k {tuple(k.shape)} v {tuple(v.shape)}")
    scale = 1.0 / math.sqrt(d) if scale is None else scale
    o = torch.empty((b, hq, s, d), dtype=torch.bfloat16, device=q.device) if out is None else out
    lse = torch.empty((b, hq, s), dtype=torch.float32, device=q.device)
    ev = LOG.begin("attn_fwd")
    rc = lib.autosp_attn_fwd(_attn_tensor(q, "q"), _attn_tensor(k, "k"), _attn_tensor(v, "v"),
                             _attn_tensor(o, "o"), lse.data_ptr(), b, hq, hkv, s, d,
                             float(scale), int(causal), _stream())
    _lib.check(rc, "attn_fwd")
    LOG.end("attn_fwd", ev, 1, causal_attn_flops(b, hq, s, d, causal))
    return o, lse


def attn_fwd_push(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, o: torch.Tensor | None,
                  lse: torch.Tensor, scale: float, causal: bool, world: int, rank: int,
                  dst_offset: int, dst_strides: tuple[int, int, int], peer_base: list[int],
                  peer_flags: list[int], epoch: int) -> int:
    """Fused K3 + K2 (autosp_attn_fwd_push): attention into o/lse AND every output row
    pushed to its token owner's receive region (head->seq all-to-all from the epilogue).
    dst_strides are the (b, s, h) element strides of the token-major destination."""
    lib = _lib.load()
    b, hq, s, d = q.shape
    hkv = k.shape[1]
    pb = (C.c_void_p * world)(*peer_base)
    pf = (C.c_void_p * world)(*peer_flags)
    spec = _lib.PushSpec(world, rank, dst_offset, dst_strides[0], dst_strides[1], dst_strides[2],
                         C.cast(pb, C.c_void_p), C.cast(pf, C.c_void_p), epoch & 0xFFFFFFFF)
    ev = LOG.begin("attn_fwd")
    o_t = _attn_tensor(o, "o") if o is not None else _lib.AttnTensor(None, 0, 0, 0)
    rc = lib.autosp_attn_fwd_push(_attn_tensor(q, "q"), _attn_tensor(k, "k"),
                                  _attn_tensor(v, "v"), o_t, lse.data_ptr(), b,
                                  hq, hkv, s, d, float(scale), int(causal), C.byref(spec),
                                  _stream())
    _lib.check(rc, "attn_fwd_push")
    LOG.end("attn_fwd", ev, 2 if world > 1 else 1, causal_attn_flops(b, hq, s, d, causal))
    return int(lib.autosp_push_check(C.byref(spec), hq))


BWD_WORKSPACE_BYTES = 1 << 30  # larger fp32 workspaces: the backward runs per kv-head group


def attn_bwd(q, k, v, o, do, lse, causal: bool = True, scale: float | None = None,
             dq=None, dk=None, dv=None, delta: torch.Tensor | None = None):
    """Flash attention backward recomputing P from the saved LSE.
    Returns (dq, dk, dv) in bf16 ([b, h, s, d]).  With `delta` ([b, hq, s] fp32 =
    rowsum(dO * O)) `o` is not read and may be None (autosp_attn_bwd_delta).
    Long sequences: the fp32 dQ accumulator workspace grows as b*hq*s*d*4 bytes (3.8 GB
    for 32 heads x 224K tokens at d = 128), so when it would exceed BWD_WORKSPACE_BYTES the
    kernels run per group of kv heads (their q heads with them) on head slices of the same
    tensors -- identical results, a fraction of the transient memory at the backward's
    memory peak."""
    lib = _lib.load()
    b, hq, s, d = q.shape
    hkv = k.shape[1]
    scale = 1.0 / math.sqrt(d) if scale is None else scale
    dev = q.device
    dq = torch.empty((b, hq, s, d), dtype=torch.bfloat16, device=dev) if dq is None else dq
    dk = torch.empty((b, hkv, s, d), dtype=torch.bfloat16, device=dev) if dk is None else dk
    dv = torch.empty((b, hkv, s, d), dtype=torch.bfloat16, device=dev) if dv is None else dv
    ws_total = lib.autosp_attn_bwd_workspace_bytes(b, hq, hkv, s, d)
    if ws_total > BWD_WORKSPACE_BYTES and hkv > 1:
        n = 1
        while n < hkv and (hkv % (2 * n) == 0) and ws_total // n > BWD_WORKSPACE_BYTES:
            n *= 2
        if n > 1:
            gk, gq = hkv // n, hq // n
            for i in range(n):
                kv, qh = slice(i * gk, (i + 1) * gk), slice(i * gq, (i + 1) * gq)
                attn_bwd(q[:, qh], k[:, kv], v[:, kv], None if o is None else o[:, qh],
                         do[:, qh], lse[:, qh].contiguous(), causal, scale,
                         dq[:, qh], dk[:, kv], dv[:, kv],
                         None if delta is None else delta[:, qh].contiguous())
            return dq, dk, dv
    ws = torch.empty(lib.autosp_attn_bwd_workspace_bytes(b, hq, hkv, s, d), dtype=torch.uint8,
                     device=dev)
    if not lse.is_contiguous() or lse.dtype != torch.float32:
        raise ValidationError("attn_bwd: lse must be contiguous fp32 [b, hq, s]")
    ev = LOG.begin("attn_bwd")
    if delta is None:
        rc = lib.autosp_attn_bwd(_attn_tensor(q, "q"), _attn_tensor(k, "k"), _attn_tensor(v, "v"),
                                 _attn_tensor(o, "o"), _attn_tensor(do, "do"), lse.data_ptr(),
                                 _attn_tensor(dq, "dq"), _attn_tensor(dk, "dk"),
                                 _attn_tensor(dv, "dv"), ws.data_ptr(), b, hq, hkv, s, d,
                                 float(scale), int(causal), _stream())
    else:
        if delta.dtype != torch.float32 or not delta.is_contiguous() or \
                tuple(delta.shape) != (b, hq, s):
            raise ValidationError("attn_bwd: delta must be contiguous fp32 [b, hq, s]")
        rc = lib.autosp_attn_bwd_delta(_attn_tensor(q, "q"), _attn_tensor(k, "k"),
                                       _attn_tensor(v, "v"), delta.data_ptr(),
                                       _attn_tensor(do, "do"), lse.data_ptr(),
                                       _attn_tensor(dq, "dq"), _attn_tensor(dk, "dk"),
                                       _attn_tensor(dv, "dv"), ws.data_ptr(), b, hq, hkv, s, d,
                                       float(scale), int(causal), _stream())
    _lib.check(rc, "attn_bwd")
    LOG.end("attn_bwd", ev, 3, 2.5 * causal_attn_flops(b, hq, s, d, causal))
    return dq, dk, dv


def attn_bwd_push(q, k, v, do, lse, delta, scale: float, causal: bool, world: int, rank: int,
                  dst_offset: int, dst_strides: tuple[int, int, int], peer_base: list[int],
                  peer_flags: list[int], epoch: int) -> int:
    """K4 fused with the head->seq all-to-all of its gradients (autosp_attn_bwd_push): no
    local dq/dk/dv; every row lands in the token owner's packed [b, s/P, H3, d] QKV
    gradient (dst_strides = its (b, s, h) element strides).  Returns the check word."""
    lib = _lib.load()
    b, hq, s, d = q.shape
    hkv = k.shape[1]
    if lse.dtype != torch.float32 or not lse.is_contiguous() or \
            delta.dtype != torch.float32 or not delta.is_contiguous() or \
            tuple(delta.shape) != (b, hq, s):
        raise ValidationError("attn_bwd_push: lse / delta must be contiguous fp32 [b, hq, s]")
    ws = torch.empty(lib.autosp_attn_bwd_workspace_bytes(b, hq, hkv, s, d), dtype=torch.uint8,
                     device=q.device)
    pb = (C.c_void_p * world)(*peer_base)
    pf = (C.c_void_p * world)(*peer_flags)
    spec = _lib.PushSpec(world, rank, dst_offset, dst_strides[0], dst_strides[1], dst_strides[2],
                         C.cast(pb, C.c_void_p), C.cast(pf, C.c_void_p), epoch & 0xFFFFFFFF)
    ev = LOG.begin("attn_bwd")
    rc = lib.autosp_attn_bwd_push(_attn_tensor(q, "q"), _attn_tensor(k, "k"), _attn_tensor(v, "v"),
                                  delta.data_ptr(), _attn_tensor(do, "do"), lse.data_ptr(),
                                  ws.data_ptr(), b, hq, hkv, s, d, float(scale), int(causal),
                                  C.byref(spec), _stream())
    _lib.check(rc, "attn_bwd_push")
    LOG.end("attn_bwd", ev, 4 if world > 1 else 3, 2.5 * causal_attn_flops(b, hq, s, d, causal))
    return int(lib.autosp_push_check(C.byref(spec), hq + 2 * hkv))


def qkv_gemm(x: torch.Tensor, w: torch.Tensor, hq: int, hkv: int, s_loc: int,
             y: torch.Tensor | None = None, pos: torch.Tensor | None = None,
             theta: float = 0.0, dst3: list | None = None, world: int = 1, rank: int = 0,
             peer_base: list[int] | None = None, peer_flags: list[int] | None = None,
             epoch: int = 0) -> torch.Tensor | int:
    """K0 (autosp_qkv_gemm): x [M, K] bf16 (rows = b * s_loc tokens), w [N, K] with
    N = (hq + 2hkv) * d.  dst3 None: plain GEMM into y [M, N] (returned).  dst3 = three
    a2a descriptors (q, k, v destinations, head-major [b, h/P, S, d]): the epilogue rounds,
    RoPE-rotates q/k rows (pos/theta) and pushes them to their head owners; returns the
    call's check word (for a2a_wait)."""
    lib = _lib.load()
    M, K = x.shape
    N = w.shape[0]
    d = N // (hq + 2 * hkv)
    if x.dtype != torch.bfloat16 or w.dtype != torch.bfloat16 or x.stride(1) != 1 or \
            w.stride(1) != 1 or w.shape[1] != K or N != (hq + 2 * hkv) * d:
        raise ValidationError("qkv_gemm: bf16 x [M, K] and w [(hq+2hkv)*d, K], rows contiguous")
    posp = 0
    if pos is not None:
        if pos.dtype != torch.float32 or not pos.is_contiguous() or not pos.is_cuda:
            raise ValidationError("qkv_gemm: positions must be a contiguous CUDA fp32 tensor")
        posp = pos.data_ptr()
    ev = LOG.begin("qkv_gemm")
    if dst3 is None:
        y = torch.empty((M, N), dtype=torch.bfloat16, device=x.device) if y is None else y
        rc = lib.autosp_qkv_gemm(x.data_ptr(), x.stride(0), w.data_ptr(), w.stride(0), M, K, hq,
                                 hkv, d, s_loc, posp or None, float(theta), 0, y.data_ptr(),
                                 y.stride(0), None, 1, 0, None, None, 0, _stream())
        _lib.check(rc, "qkv_gemm")
        LOG.end("qkv_gemm", ev, 1, 2.0 * M * N * K)
        return y
    arr = (_lib.A2ATensor * 3)(*dst3)
    pb = (C.c_void_p * world)(*peer_base)
    pf = (C.c_void_p * world)(*peer_flags)
    rc = lib.autosp_qkv_gemm(x.data_ptr(), x.stride(0), w.data_ptr(), w.stride(0), M, K, hq, hkv,
                             d, s_loc, posp or None, float(theta), int(pos is not None), None, 0,
                             arr, world, rank, pb, pf, epoch & 0xFFFFFFFF, _stream())
    _lib.check(rc, "qkv_gemm")
    LOG.end("qkv_gemm", ev, 2 if world > 1 else 1, 2.0 * M * N * K)
    return a2a_check(_lib.SEQ_TO_HEAD, list(dst3))


# ----------------------------------------------------------------------------- all-to-all
def a2a_tensor_desc(src: torch.Tensor, heads: int, dst_offset: int,
                    dst_strides: tuple[int, int, int], rope: bool = False) -> _lib.A2ATensor:
    """src is a logical [b, s, h, d] view with d contiguous."""
    if src.dim() != 4 or src.stride(3) != 1:
        raise ValidationError("a2a source must be a [b, s, h, d] view with contiguous head_dim")
    sb, ss, sh, _ = src.stride()
    db, ds, dh = dst_strides
    return _lib.A2ATensor(src.data_ptr(), sb, ss, sh, dst_offset, db, ds, dh, heads, int(rope))


def a2a_launch(direction: int, descs: list, b: int, s_global: int, d: int, elem_bytes: int,
               world: int, rank: int, peer_base: list[int], peer_flags: list[int],
               epoch: int, pos: torch.Tensor | None = None, theta: float = 0.0) -> int:
    """K1/K2.  With `pos` (fp32 positions of the source tokens) the descriptors flagged
    rope are rotated on the way (autosp_a2a_rope).  Returns the call's check word."""
    lib = _lib.load()
    arr = (_lib.A2ATensor * len(descs))(*descs)
    pb = (C.c_void_p * world)(*peer_base)
    pf = (C.c_void_p * world)(*peer_flags)
    ev = LOG.begin("a2a")
    if pos is None:
        rc = lib.autosp_a2a(direction, arr, len(descs), b, s_global, d, elem_bytes, world, rank,
                            pb, pf, epoch & 0xFFFFFFFF, _stream())
    else:
        if pos.dtype != torch.float32 or not pos.is_contiguous() or not pos.is_cuda:
            raise ValidationError("a2a rope positions must be a contiguous CUDA fp32 tensor")
        rc = lib.autosp_a2a_rope(direction, arr, len(descs), b, s_global, d, elem_bytes, world,
                                 rank, pb, pf, epoch & 0xFFFFFFFF, pos.data_ptr(), float(theta),
                                 _stream())
    _lib.check(rc, "a2a")
    # bytes sent to peers = (P-1)/P of this rank's local share of every tensor
    local = sum(b * s_global * dsc.heads * d * elem_bytes for dsc in descs) // max(world, 1)
    LOG.end("a2a", ev, 2 if world > 1 else 1, nbytes=local * (world - 1) / max(world, 1))
    return a2a_check(direction, descs)


def a2a_grad_out(do_desc, o_desc, b: int, s_global: int, d: int, world: int, rank: int,
                 peer_base: list[int], peer_flags: list[int], epoch: int) -> int:
    """autosp_a2a_grad_out: dO reshard seq->head fused with delta = rowsum(dO * O) (o_desc's
    destination is the fp32 delta).  Returns the check word."""
    lib = _lib.load()
    arr = (_lib.A2ATensor * 2)(do_desc, o_desc)
    pb = (C.c_void_p * world)(*peer_base)
    pf = (C.c_void_p * world)(*peer_flags)
    ev = LOG.begin("a2a")
    rc = lib.autosp_a2a_grad_out(arr, b, s_global, d, world, rank, pb, pf, epoch & 0xFFFFFFFF,
                                 _stream())
    _lib.check(rc, "a2a_grad_out")
    local = b * s_global * do_desc.heads * d * 2 // max(world, 1)
    LOG.end("a2a", ev, 2 if world > 1 else 1,
            nbytes=(local + local // (2 * d) * 4) * (world - 1) / max(world, 1))
    return a2a_check(_lib.SEQ_TO_HEAD, [do_desc, o_desc])


def a2a_check(direction: int, descs: list) -> int:
    """Check word of a call with these destination descriptors (what autosp_a2a_wait
    compares against every sender's own view)."""
    arr = (_lib.A2ATensor * len(descs))(*descs)
    return int(_lib.load().autosp_a2a_check(direction, arr, len(descs)))


def a2a_wait(local_flags: int, world: int, rank: int, epoch: int, check: int) -> None:
    """Wait for every peer's arrival of `epoch`; `check` = this rank's check word of the
    call (a2a_launch's / attn_fwd_push's return value)."""
    rc = _lib.load().autosp_a2a_wait(local_flags, world, rank, epoch & 0xFFFFFFFF,
                                     check & 0xFFFFFFFF, _stream())
    _lib.check(rc, "a2a_wait")
    LOG.end("a2a_wait", None, 1 if world > 1 else 0)


def a2a_mark_ready(flags: list[int], epoch: int) -> None:
    pf = (C.c_void_p * len(flags))(*flags)
    rc = _lib.load().autosp_a2a_mark_ready(pf, len(flags), epoch & 0xFFFFFFFF, _stream())
    _lib.check(rc, "a2a_mark_ready")


def a2a_loopback(direction: str, shards: list[torch.Tensor]) -> list[torch.Tensor]:
    """Run the push kernel for P VIRTUAL ranks on one GPU (each rank's receive region and
    flag block is a local allocation).  Same semantics as the reference's
    all_to_all_shards (executor.py:203-230); used by tests and the single-GPU bench."""
    P = len(shards)
    b, s_src, h_src, d = shards[0].shape
    dev, dt = shards[0].device, shards[0].dtype
    eb = shards[0].element_size()
    if direction == "seq_to_head":
        out_shape = (b, s_src * P, h_src // P, d)
        dirn, s_glob = _lib.SEQ_TO_HEAD, s_src * P
    elif direction == "head_to_seq":
        out_shape = (b, s_src // P, h_src * P, d)
        dirn, s_glob = _lib.HEAD_TO_SEQ, s_src
    else:
        raise ValidationError(f"unknown all-to-all direction {direction!r}")
    outs = [torch.empty(out_shape, dtype=dt, device=dev) for _ in range(P)]
    flags = torch.zeros((P, _lib.FLAG_WORDS), dtype=torch.int32, device=dev)
    fptr = [flags[j].data_ptr() for j in range(P)]
    optr = [o.data_ptr() for o in outs]
    ostr = outs[0].stride()
    a2a_mark_ready(fptr, 1)
    for r in range(P):
        desc = a2a_tensor_desc(shards[r], h_src, 0, (ostr[0], ostr[1], ostr[2]))
        chk = a2a_launch(dirn, [desc], b, s_glob, d, eb, P, r, optr, fptr, 1)
    for r in range(P):
        a2a_wait(fptr[r], P, r, 1, chk)
    return outs


# ----------------------------------------------------------------------------- fused elementwise
def _bf16_rows(t: torch.Tensor, name: str) -> int:
    if not t.is_cuda or t.dtype != torch.bfloat16 or t.stride(-1) != 1:
        raise ValidationError(f"{name}: expected a CUDA bf16 tensor with contiguous last dim")
    return t.stride(-2) if t.dim() >= 2 else t.shape[-1]


def swiglu_fwd(gu: torch.Tensor) -> torch.Tensor:
    """gu [..., 2F] -> silu(gu[..., :F]) * gu[..., F:]."""
    g2 = gu.reshape(-1, gu.shape[-1])
    F = g2.shape[1] // 2
    out = torch.empty(g2.shape[0], F, dtype=gu.dtype, device=gu.device)
    rc = _lib.load().autosp_swiglu_fwd(g2.data_ptr(), out.data_ptr(), g2.shape[0], F,
                                       _bf16_rows(g2, "gu"), F, _stream())
    _lib.check(rc, "swiglu_fwd")
    LOG.end("swiglu", None, 1)
    return out.view(*gu.shape[:-1], F)


def swiglu_bwd(gu: torch.Tensor, dout: torch.Tensor) -> torch.Tensor:
    g2 = gu.reshape(-1, gu.shape[-1])
    d2 = dout.reshape(-1, dout.shape[-1])
    if d2.stride(-1) != 1:
        d2 = d2.contiguous()
    F = g2.shape[1] // 2
    dgu = torch.empty_like(g2)
    rc = _lib.load().autosp_swiglu_bwd(g2.data_ptr(), d2.data_ptr(), dgu.data_ptr(), g2.shape[0],
                                       F, _bf16_rows(g2, "gu"), _bf16_rows(d2, "dout"),
                                       dgu.stride(0), _stream())
    _lib.check(rc, "swiglu_bwd")
    LOG.end("swiglu", None, 1)
    return dgu.view(gu.shape)


def rope(x: torch.Tensor, pos: torch.Tensor, theta: float, inverse: bool = False) -> torch.Tensor:
    """x [b, s, h, d] (strided view, d contiguous) -> rotated contiguous [b, s, h, d]."""
    if x.stride(-1) != 1 or x.dtype != torch.bfloat16 or not x.is_cuda:
        raise ValidationError("rope: CUDA bf16 [b, s, h, d] view with contiguous d required")
    b, s, h, d = x.shape
    y = torch.empty((b, s, h, d), dtype=x.dtype, device=x.device)
    pos = pos.to(torch.float32).contiguous()
    rc = _lib.load().autosp_rope(x.data_ptr(), y.data_ptr(), b, s, h, d, x.stride(0), x.stride(1),
                                 x.stride(2), y.stride(0), y.stride(1), y.stride(2),
                                 pos.data_ptr(), float(theta), int(inverse), _stream())
    _lib.check(rc, "rope")
    LOG.end("rope", None, 1)
    return y


def rope_segments(pairs: list[tuple[torch.Tensor, torch.Tensor, bool]], pos: torch.Tensor,
                  theta: float, inverse: bool = False) -> None:
    """One launch over up to 3 (src, dst, rotate) [b, s, h, d] view pairs (d contiguous):
    dst = RoPE(src) when rotate else src."""
    segs = []
    b, s, _, d = pairs[0][0].shape
    for src, dst, rot in pairs:
        for t, n in ((src, "src"), (dst, "dst")):
            if t.stride(-1) != 1 or t.dtype != torch.bfloat16 or not t.is_cuda:
                raise ValidationError(f"rope_segments: {n} must be a CUDA bf16 view, d contiguous")
        if src.shape != dst.shape or src.shape[0] != b or src.shape[1] != s:
            raise ValidationError("rope_segments: src/dst shape mismatch")
        segs.append(_lib.RopeSegment(src.data_ptr(), dst.data_ptr(), src.stride(0), src.stride(1),
                                     src.stride(2), dst.stride(0), dst.stride(1), dst.stride(2),
                                     src.shape[2], int(rot)))
    arr = (_lib.RopeSegment * len(segs))(*segs)
    pos = pos.to(torch.float32).contiguous()
    rc = _lib.load().autosp_rope_segments(arr, len(segs), b, s, d, pos.data_ptr(), float(theta),
                                          int(inverse), _stream())
    _lib.check(rc, "rope_segments")
    LOG.end("rope", None, 1)


def _rows2d(t: torch.Tensor, name: str) -> torch.Tensor:
    t2 = t.reshape(-1, t.shape[-1])
    if not t2.is_cuda or t2.dtype != torch.bfloat16 or t2.stride(-1) != 1:
        raise ValidationError(f"{name}: expected a CUDA bf16 tensor with contiguous last dim")
    return t2


def rms_norm_fwd(x: torch.Tensor, w: torch.Tensor, eps: float):
    """RMSNorm over the last dim: (y bf16 like x, rstd fp32 [rows])."""
    x2 = _rows2d(x, "x")
    rows, d = x2.shape
    y = torch.empty((rows, d), dtype=x.dtype, device=x.device)
    rstd = torch.empty(rows, dtype=torch.float32, device=x.device)
    w = w.contiguous()
    rc = _lib.load().autosp_rms_norm_fwd(x2.data_ptr(), w.data_ptr(), y.data_ptr(),
                                         rstd.data_ptr(), rows, d, x2.stride(0), d, float(eps),
                                         _stream())
    _lib.check(rc, "rms_norm_fwd")
    LOG.end("rms_norm", None, 1)
    return y.view(x.shape), rstd.view(x.shape[:-1])


def rms_norm_bwd(dy: torch.Tensor, x: torch.Tensor, w: torch.Tensor, rstd: torch.Tensor):
    """(dx like x, dw like w) in one pass over (dy, x)."""
    lib = _lib.load()
    d2 = _rows2d(dy if dy.stride(-1) == 1 else dy.contiguous(), "dy")
    x2 = _rows2d(x, "x")
    rows, d = x2.shape
    dx = torch.empty((rows, d), dtype=x.dtype, device=x.device)
    dw = torch.empty(d, dtype=w.dtype, device=w.device)
    ws = torch.empty(lib.autosp_rms_norm_bwd_workspace_bytes(d), dtype=torch.uint8,
                     device=x.device)
    rs = rstd.reshape(-1).contiguous()
    w = w.contiguous()
    rc = lib.autosp_rms_norm_bwd(d2.data_ptr(), x2.data_ptr(), w.data_ptr(), rs.data_ptr(),
                                 dx.data_ptr(), dw.data_ptr(), ws.data_ptr(), rows, d,
                                 d2.stride(0), x2.stride(0), d, _stream())
    _lib.check(rc, "rms_norm_bwd")
    LOG.end("rms_norm", None, 2)
    return dx.view(x.shape), dw


def ce_fwd(logits: torch.Tensor, labels: torch.Tensor):
    """Row-wise (lse, loss) of bf16 logits [n, V] (leading dim may exceed V)."""
    n, V = logits.shape
    lse = torch.empty(n, dtype=torch.float32, device=logits.device)
    loss = torch.empty(n, dtype=torch.float32, device=logits.device)
    labels = labels.to(torch.int64).contiguous()
    rc = _lib.load().autosp_ce_fwd(logits.data_ptr(), labels.data_ptr(), lse.data_ptr(),
                                   loss.data_ptr(), n, V, _bf16_rows(logits, "logits"), _stream())
    _lib.check(rc, "ce_fwd")
    LOG.end("ce", None, 1)
    return lse, loss


def ce_bwd_(logits: torch.Tensor, labels: torch.Tensor, lse: torch.Tensor, g: float) -> torch.Tensor:
    """In place: logits <- g * (softmax(logits) - onehot(labels))."""
    n, V = logits.shape
    labels = labels.to(torch.int64).contiguous()
    rc = _lib.load().autosp_ce_bwd(logits.data_ptr(), labels.data_ptr(), lse.data_ptr(), float(g),
                                   n, V, _bf16_rows(logits, "logits"), _stream())
    _lib.check(rc, "ce_bwd")
    LOG.end("ce", None, 1)
    return logits
