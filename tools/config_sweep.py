"""Per-rank work of every BASELINE.json configuration at full size, on ONE B200: the
attention kernels (K3 fwd, K4 bwd) on the heads a rank owns after the seq->head reshard
(hq/P q heads, hkv/P kv heads, the whole sequence) and the reshard kernel with P virtual
ranks (loopback).  Prints one JSON line per config (TF/s, ms per layer, projected
attention share of the per-rank step).  Evidence for the multi-GPU configs that this
single-GPU round cannot run end to end."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2604_27089_b200 import kernels as K

CONFIGS = [  # name, P, hq, hkv, d, s, layers
    ("C2 llama3.2-1b 32K SP=8", 8, 32, 8, 64, 32768, 16),
    ("C3 llama3-8b 128K SP=8", 8, 32, 8, 128, 131072, 32),
    ("C5 llama3-8b GQA 256K SP=8", 8, 32, 8, 128, 262144, 32),
    ("C4 llama3-8b 512K SP=8", 8, 32, 8, 128, 524288, 32),
]


_pk = Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json"
PEAK = json.loads(_pk.read_text()).get("bf16_tflops_sustained", 1400.0) if _pk.exists() else 1400.0


def timed(fn, iters):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


for name, P, hq, hkv, d, s, L in CONFIGS:
    ql, kl = hq // P, hkv // P
    q = torch.randn(1, ql, s, d, device="cuda").bfloat16()
    k = torch.randn(1, kl, s, d, device="cuda").bfloat16()
    v = torch.randn(1, kl, s, d, device="cuda").bfloat16()
    do = torch.randn(1, ql, s, d, device="cuda").bfloat16()
    o, lse = K.attn_fwd(q, k, v)
    it = 3 if s >= 262144 else 10
    tf = timed(lambda: K.attn_fwd(q, k, v, out=o), it)
    tb = timed(lambda: K.attn_bwd(q, k, v, o, do, lse), it)
    fl = K.causal_attn_flops(1, ql, s, d)
    # reshard of one layer's q/k/v (seq->head), P virtual ranks on this GPU
    shards = [torch.randn(1, s // P, hq + 2 * hkv, d, device="cuda").bfloat16() for _ in range(P)]
    ta = timed(lambda: K.a2a_loopback("seq_to_head", shards), 3)
    per_rank_bytes = (s // P) * (hq + 2 * hkv) * d * 2
    print(json.dumps({
        "config": name, "per_rank_heads": [ql, kl], "seq": s, "head_dim": d,
        "attn_fwd_ms_per_layer": tf, "attn_fwd_tflops": fl / tf / 1e9,
        "attn_bwd_ms_per_layer": tb, "attn_bwd_tflops": 2.5 * fl / tb / 1e9,
        "attn_fwd_frac_of_sustained_peak": fl / tf / 1e9 / PEAK,
        "attn_bwd_frac_of_sustained_peak": 2.5 * fl / tb / 1e9 / PEAK,
        "attention_ms_per_step": L * (tf + tb),
        "a2a_qkv_loopback_ms_all_ranks": ta, "a2a_bytes_sent_per_rank": per_rank_bytes,
        "a2a_nvlink_model_ms": per_rank_bytes * (P - 1) / P / 770e9 * 1e3}), flush=True)
    del q, k, v, do, o, lse, shards
    torch.cuda.empty_cache()
