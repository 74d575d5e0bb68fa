"""K0, the tcgen05 QKV-projection GEMM with the seq->head all-to-all in its epilogue
(autosp_qkv_gemm):

1. as a plain GEMM it matches an fp32 torch reference within bf16 output rounding;
2. fused (RoPE + push to the head owners, P virtual ranks on one GPU through the real
   epoch protocol) it is BIT-EXACT against the unfused path "K0 as a plain GEMM -> bf16
   -> K1 RoPE push" (autosp_a2a_rope), i.e. folding the reshard into the epilogue
   changes nothing but where the bytes go (reference: Linear + all_to_all_shards
   seq_to_head, transformer.py:66-72, executor.py:203-230)."""

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("M,K,hq,hkv,d", [(256, 512, 8, 4, 64), (128, 256, 4, 2, 128),
                                         (512, 2048, 32, 8, 64), (256, 128, 8, 8, 32)])
def test_qkv_gemm_plain_matches_torch(M, K, hq, hkv, d):
    from paper_2604_27089_b200 import kernels
    g = torch.Generator().manual_seed(M + K + d)
    x = torch.randn(M, K, generator=g).bfloat16().cuda()
    w = (torch.randn((hq + 2 * hkv) * d, K, generator=g) * K ** -0.5).bfloat16().cuda()
    y = kernels.qkv_gemm(x, w, hq, hkv, s_loc=M)
    ref = x.float() @ w.float().t()
    err = float((y.float() - ref).abs().max() / ref.abs().max())
    assert err < 1e-2, err


def test_qkv_gemm_rejects_unsupported_shapes():
    from paper_2604_27089_b200 import kernels
    from paper_2604_27089_b200.errors import SeqcompError
    x = torch.zeros(100, 256, dtype=torch.bfloat16, device="cuda")
    w = torch.zeros(1024, 256, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(SeqcompError):
        kernels.qkv_gemm(x, w, 8, 4, s_loc=100)


@pytest.mark.parametrize("P,b,s_loc,K,hq,hkv,d", [(2, 1, 128, 256, 8, 4, 64),
                                                   (4, 2, 128, 512, 8, 4, 128),
                                                   (8, 1, 256, 1024, 32, 8, 64)])
def test_qkv_gemm_push_bit_exact_vs_gemm_then_k1(P, b, s_loc, K, hq, hkv, d):
    from paper_2604_27089_b200 import _lib, kernels
    S = s_loc * P
    H3 = hq + 2 * hkv
    theta = 500000.0
    g = torch.Generator().manual_seed(P * 100 + d)
    xs = [torch.randn(b * s_loc, K, generator=g).bfloat16().cuda() for _ in range(P)]
    w = (torch.randn(H3 * d, K, generator=g) * K ** -0.5).bfloat16().cuda()
    pos = [torch.arange(r * s_loc, (r + 1) * s_loc, dtype=torch.float32).cuda() for r in range(P)]
    qn, kn = b * (hq // P) * S * d, b * (hkv // P) * S * d

    def dsts(heads_list):
        out, off = [], 0
        for h in heads_list:
            hl = h // P
            out.append((off * 2, (hl * S * d, d, S * d), h))
            off += b * hl * S * d
        return out

    layout = dsts((hq, hkv, hkv))

    def run(fused):
        regions = [torch.zeros(qn + 2 * kn, dtype=torch.bfloat16, device="cuda")
                   for _ in range(P)]
        flags = torch.zeros((P, _lib.FLAG_WORDS), dtype=torch.int32, device="cuda")
        fptr = [flags[j].data_ptr() for j in range(P)]
        rptr = [x.data_ptr() for x in regions]
        kernels.a2a_mark_ready(fptr, 1)  # loopback: every virtual rank reached epoch 1
        chks = []
        for r in range(P):
            if fused:
                dst3 = [_lib.A2ATensor(None, 0, 0, 0, off, *st, h, 0) for off, st, h in layout]
                chks.append(kernels.qkv_gemm(xs[r], w, hq, hkv, s_loc, pos=pos[r], theta=theta,
                                             dst3=dst3, world=P, rank=r, peer_base=rptr,
                                             peer_flags=fptr, epoch=1))
            else:
                y = kernels.qkv_gemm(xs[r], w, hq, hkv, s_loc).view(b, s_loc, H3, d)
                srcs = (y[:, :, :hq], y[:, :, hq:hq + hkv], y[:, :, hq + hkv:])
                descs = [kernels.a2a_tensor_desc(src, h, off, st, rope=(i < 2))
                         for i, (src, (off, st, h)) in enumerate(zip(srcs, layout))]
                chks.append(kernels.a2a_launch(_lib.SEQ_TO_HEAD, descs, b, S, d, 2, P, r, rptr,
                                               fptr, 1, pos=pos[r], theta=theta))
        for r in range(P):
            kernels.a2a_wait(fptr[r], P, r, 1, chks[r])
        torch.cuda.synchronize()
        return regions

    fused, ref = run(True), run(False)
    for r in range(P):
        assert torch.equal(fused[r].view(torch.int16), ref[r].view(torch.int16)), r
    assert any(bool(x.abs().sum() > 0) for x in fused)
