"""GPU numerics of the fused layer kernels (csrc/fused.cu) against plain PyTorch fp32
references of the same ops, and of the fused Llama block against the unfused one."""

import math

import pytest
import torch
import torch.nn.functional as F

pytestmark = pytest.mark.gpu
TOL = 2e-2  # max|a - ref| / max|ref|, bf16 outputs


def _rel(a, b):
    a, b = a.float(), b.float()
    return float((a - b).abs().max() / b.abs().max().clamp_min(1e-30))


@pytest.fixture(scope="module", autouse=True)
def _lib():
    from paper_2604_27089_b200 import _build, _lib
    _build.build()
    _lib.load()


@pytest.mark.parametrize("rows,ffn", [(1, 8), (37, 64), (512, 8192)])
def test_swiglu_fwd_bwd(rows, ffn):
    from paper_2604_27089_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(rows)
    gu = torch.randn(rows, 2 * ffn, device="cuda", generator=g).bfloat16().requires_grad_(True)
    dout = torch.randn(rows, ffn, device="cuda", generator=g).bfloat16()
    y = ops.swiglu(gu)
    y.backward(dout)
    ref_in = gu.detach().float().requires_grad_(True)
    a, b = ref_in.chunk(2, dim=-1)
    ref = F.silu(a) * b
    ref.backward(dout.float())
    assert _rel(y, ref) < TOL
    assert _rel(gu.grad, ref_in.grad) < TOL


def _rope_ref(x, pos, theta):
    d = x.shape[-1]
    inv = 1.0 / (theta ** (torch.arange(0, d, 2, device=x.device, dtype=torch.float64) / d))
    fr = pos.double()[:, None] * inv[None, :]
    c, s = fr.cos()[None, :, None, :], fr.sin()[None, :, None, :]
    x1, x2 = x[..., : d // 2].double(), x[..., d // 2:].double()
    return torch.cat((x1 * c - x2 * s, x2 * c + x1 * s), dim=-1)


@pytest.mark.parametrize("b,s,h,d,off", [(1, 64, 4, 64, 0), (2, 33, 3, 128, 4096),
                                          (1, 256, 8, 64, 131072)])
def test_rope_fwd_bwd_with_rank_offset(b, s, h, d, off):
    from paper_2604_27089_b200 import ops
    theta = 500000.0
    full = torch.randn(b, s, h + 2, d, device="cuda").bfloat16()
    x = full[:, :, 1:h + 1].requires_grad_(False)  # strided view, like q inside qkv
    xr = x.clone().requires_grad_(True)
    pos = torch.arange(off, off + s, device="cuda").float()
    y = ops.rope(xr, pos, theta, False)
    ref = _rope_ref(x, pos, theta)
    assert _rel(y, ref) < TOL
    dy = torch.randn_like(y)
    y.backward(dy)
    # rotation is orthogonal: dx = R(-angle) dy
    assert _rel(xr.grad, _rope_ref(dy, pos, theta) * 0 + _inv_rot(dy, pos, theta)) < TOL
    back = ops.rope(y.detach(), pos, theta, True)
    assert _rel(back, x) < TOL


def _inv_rot(dy, pos, theta):
    d = dy.shape[-1]
    inv = 1.0 / (theta ** (torch.arange(0, d, 2, device=dy.device, dtype=torch.float64) / d))
    fr = pos.double()[:, None] * inv[None, :]
    c, s = fr.cos()[None, :, None, :], fr.sin()[None, :, None, :]
    y1, y2 = dy[..., : d // 2].double(), dy[..., d // 2:].double()
    return torch.cat((y1 * c + y2 * s, y2 * c - y1 * s), dim=-1)


@pytest.mark.parametrize("n,V", [(3, 64), (17, 1000), (256, 128256)])
def test_cross_entropy_fwd_bwd(n, V):
    from paper_2604_27089_b200 import kernels
    g = torch.Generator(device="cuda").manual_seed(V)
    logits = (torch.randn(n, V, device="cuda", generator=g) * 3).bfloat16()
    labels = torch.randint(0, V, (n,), device="cuda", generator=g)
    lse, loss = kernels.ce_fwd(logits, labels)
    ref_lse = torch.logsumexp(logits.float(), -1)
    ref_loss = F.cross_entropy(logits.float(), labels, reduction="none")
    assert float((lse - ref_lse).abs().max()) < 1e-3 * max(1.0, float(ref_lse.abs().max()))
    assert float((loss - ref_loss).abs().max()) < 1e-3 * max(1.0, float(ref_loss.abs().max()))
    lf = logits.float().requires_grad_(True)
    F.cross_entropy(lf, labels, reduction="sum").mul(0.5).backward()
    dl = kernels.ce_bwd_(logits.clone(), labels, lse, 0.5)
    assert _rel(dl, lf.grad) < TOL


def test_cross_entropy_ignores_out_of_range_labels():
    """labels outside [0, vocab) (-100 padding, >= vocab) contribute 0 to the
    loss and get an all-zero gradient row (torch ignore_index with reduction='sum')."""
    from paper_2604_27089_b200 import kernels
    from paper_2604_27089_b200.workloads import lm_loss
    n, V = 9, 1000
    g = torch.Generator(device="cuda").manual_seed(1)
    logits = (torch.randn(n, V, device="cuda", generator=g) * 3).bfloat16()
    labels = torch.randint(0, V, (n,), device="cuda", generator=g)
    labels[0], labels[4], labels[8] = -100, V, -1
    lse, loss = kernels.ce_fwd(logits, labels)
    ref = F.cross_entropy(logits.float(), labels.masked_fill((labels < 0) | (labels >= V), -100),
                          reduction="none", ignore_index=-100)
    assert float((loss - ref).abs().max()) < 1e-3 * max(1.0, float(ref.abs().max()))
    assert float(loss[0]) == 0.0 and float(loss[4]) == 0.0 and float(loss[8]) == 0.0
    dl = kernels.ce_bwd_(logits.clone(), labels, lse, 1.0)
    assert not dl[[0, 4, 8]].float().abs().any()
    # through the chunked LM loss (chunk boundary inside the batch)
    h = torch.randn(n, 64, device="cuda", generator=g).bfloat16().requires_grad_(True)
    w = (torch.randn(V, 64, device="cuda", generator=g) * 0.1).bfloat16().requires_grad_(True)
    tot = lm_loss(h, w, labels, chunk=4)
    hf, wf = h.detach().float().requires_grad_(True), w.detach().float().requires_grad_(True)
    lab = labels.masked_fill((labels < 0) | (labels >= V), -100)
    rf = F.cross_entropy(hf @ wf.t(), lab, reduction="sum", ignore_index=-100)
    tot.backward()
    rf.backward()
    assert abs(float(tot) - float(rf)) < 1e-2 * abs(float(rf))
    assert not h.grad[[0, 4, 8]].float().abs().any()
    assert _rel(h.grad, hf.grad) < TOL and _rel(w.grad, wf.grad) < TOL


def test_fused_llama_block_matches_unfused():
    """Same weights, fused (autosp rope/swiglu/F.rms_norm) vs plain torch block, fwd+bwd."""
    from paper_2604_27089_b200 import ops
    from paper_2604_27089_b200.workloads import LlamaBlock, LlamaConfig
    cfg = LlamaConfig("tiny", 256, 1, 4, 2, 512, vocab=1000)
    torch.manual_seed(0)
    a = LlamaBlock(cfg, torch.bfloat16, "cuda", fused=True)
    bblk = LlamaBlock(cfg, torch.bfloat16, "cuda", fused=False)
    with torch.no_grad():
        for pa, pb in zip(a.parameters(), bblk.parameters()):
            pa.copy_(torch.randn_like(pa) * 0.05 if pa.dim() == 2 else torch.ones_like(pa))
            pb.copy_(pa)
    s = 256
    x = torch.randn(1, s, cfg.d_model, device="cuda").bfloat16()
    pos = torch.arange(s, device="cuda").float()
    inv = 1.0 / (cfg.rope_theta ** (torch.arange(0, cfg.head_dim, 2, device="cuda").float()
                                    / cfg.head_dim))
    fr = pos[:, None] * inv[None, :]
    xa = x.clone().requires_grad_(True)
    xb = x.clone().requires_grad_(True)
    ya = a(xa, None, None, pos)
    yb = bblk(xb, fr.cos(), fr.sin(), pos)
    assert _rel(ya, yb) < TOL
    dy = torch.randn_like(ya)
    ya.backward(dy)
    yb.backward(dy)
    assert _rel(xa.grad, xb.grad) < 5e-2
    for pa, pb in zip(a.parameters(), bblk.parameters()):
        assert _rel(pa.grad, pb.grad) < 5e-2


@pytest.mark.parametrize("b,s,hq,hkv,d,off", [(1, 64, 4, 2, 64, 0), (2, 40, 8, 2, 128, 4096),
                                               (1, 256, 32, 8, 64, 131072)])
def test_qkv_rope_split_and_packed_gradient(b, s, hq, hkv, d, off):
    """autosp::qkv_rope = split of the packed QKV projection + RoPE of q/k in one launch;
    its backward assembles the packed gradient (inverse rotation of dq/dk, dv copied)."""
    from paper_2604_27089_b200 import ops
    theta = 500000.0
    qkv = torch.randn(b, s, hq + 2 * hkv, d, device="cuda").bfloat16().requires_grad_(True)
    pos = torch.arange(off, off + s, device="cuda").float()
    q, k, v = ops.qkv_rope(qkv, pos, theta, hq, hkv)
    x = qkv.detach()
    assert _rel(q, _rope_ref(x[:, :, :hq], pos, theta)) < TOL
    assert _rel(k, _rope_ref(x[:, :, hq:hq + hkv], pos, theta)) < TOL
    assert torch.equal(v, x[:, :, hq + hkv:])
    dq, dk, dv = (torch.randn_like(t) for t in (q, k, v))
    torch.autograd.backward((q, k, v), (dq, dk, dv))
    g = qkv.grad
    assert _rel(g[:, :, :hq], _inv_rot(dq, pos, theta)) < TOL
    assert _rel(g[:, :, hq:hq + hkv], _inv_rot(dk, pos, theta)) < TOL
    assert torch.equal(g[:, :, hq + hkv:], dv)


@pytest.mark.parametrize("rows,d", [(1, 64), (37, 2048), (4096, 4096), (300, 1000)])
def test_rms_norm_fwd_bwd(rows, d):
    """autosp::rms_norm (reference executor.py:43-45) vs an fp32 torch reference, incl. the
    one-pass weight gradient."""
    from paper_2604_27089_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(d)
    x = (torch.randn(rows, d, device="cuda", generator=g) * 3).bfloat16().requires_grad_(True)
    w = (1 + 0.1 * torch.randn(d, device="cuda", generator=g)).bfloat16().requires_grad_(True)
    dy = torch.randn(rows, d, device="cuda", generator=g).bfloat16()
    y = ops.rms_norm(x, w, 1e-5)
    y.backward(dy)
    xr = x.detach().float().requires_grad_(True)
    wr = w.detach().float().requires_grad_(True)
    ref = xr * torch.rsqrt(xr.pow(2).mean(-1, keepdim=True) + 1e-5) * wr
    ref.backward(dy.float())
    assert _rel(y, ref) < TOL
    assert _rel(x.grad, xr.grad) < TOL
    assert _rel(w.grad, wr.grad) < TOL
