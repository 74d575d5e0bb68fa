"""CUDA-event timing of K0 (autosp_qkv_gemm) as a plain GEMM against cuBLAS (torch.matmul)
at the per-rank QKV-projection shapes of the bench models, and of the fused RoPE + push
epilogue in loopback (P virtual ranks' receive regions on one GPU) against "cuBLAS GEMM +
K1 RoPE push" -- development tool; prints one JSON line per shape."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2604_27089_b200 import _lib, kernels as K


def timeit(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


def run(name, M, Kd, hq, hkv, d, P):
    N = (hq + 2 * hkv) * d
    x = torch.randn(M, Kd, device="cuda").bfloat16()
    w = (torch.randn(N, Kd, device="cuda") * Kd ** -0.5).bfloat16()
    y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    t_k0 = timeit(lambda: K.qkv_gemm(x, w, hq, hkv, s_loc=M, y=y))
    t_cb = timeit(lambda: torch.matmul(x, w.t(), out=y))
    fl = 2.0 * M * N * Kd
    out = {"shape": name, "M": M, "N": N, "K": Kd, "k0_ms": t_k0, "k0_tflops": fl / t_k0 / 1e9,
           "cublas_ms": t_cb, "cublas_tflops": fl / t_cb / 1e9}
    # fused push (this rank = 0 of P; loopback regions) vs cuBLAS + K1
    S = M * P
    qn, kn = (hq // P) * S * d, (hkv // P) * S * d
    regions = [torch.empty(qn + 2 * kn, dtype=torch.bfloat16, device="cuda") for _ in range(P)]
    flags = torch.zeros((P, _lib.FLAG_WORDS), dtype=torch.int32, device="cuda")
    fptr, rptr = [flags[j].data_ptr() for j in range(P)], [r.data_ptr() for r in regions]
    pos = torch.arange(M, dtype=torch.float32, device="cuda")
    lay, off = [], 0
    for h in (hq, hkv, hkv):
        lay.append((off * 2, ((h // P) * S * d, d, S * d), h))
        off += (h // P) * S * d
    ep = [0]

    def fused():
        ep[0] += 1
        K.a2a_mark_ready(fptr, ep[0])
        dst3 = [_lib.A2ATensor(None, 0, 0, 0, o, *st, h, 0) for o, st, h in lay]
        K.qkv_gemm(x, w, hq, hkv, M, pos=pos, theta=5e5, dst3=dst3, world=P, rank=0,
                   peer_base=rptr, peer_flags=fptr, epoch=ep[0])

    def unfused():
        ep[0] += 1
        K.a2a_mark_ready(fptr, ep[0])
        torch.matmul(x, w.t(), out=y)
        yv = y.view(1, M, hq + 2 * hkv, d)
        srcs = (yv[:, :, :hq], yv[:, :, hq:hq + hkv], yv[:, :, hq + hkv:])
        descs = [K.a2a_tensor_desc(s, h, o, st, rope=(i < 2))
                 for i, (s, (o, st, h)) in enumerate(zip(srcs, lay))]
        K.a2a_launch(_lib.SEQ_TO_HEAD, descs, 1, S, d, 2, P, 0, rptr, fptr, ep[0], pos=pos,
                     theta=5e5)

    out["fused_push_ms"] = timeit(fused)
    out["cublas_plus_k1_ms"] = timeit(unfused)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    for P in (8, 4, 2):
        run(f"llama3.2-1b 32K P={P}", 32768 // P, 2048, 32, 8, 64, P)
    run("llama3-8b 128K P=8", 16384, 4096, 32, 8, 128, 8)
    run("llama3.2-1b 32K P=1 (plain)", 32768, 2048, 32, 8, 64, 2)
