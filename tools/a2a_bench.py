"""Single-GPU measurement of the all-to-all push kernel (K1/K2) in loopback: P virtual
ranks whose receive regions are local allocations, driven through the real C ABI
(handshake + push + wait kernels, epoch flags).  Reports per-call time and the kernel's
HBM rate (bytes read + written) against the measured copy bandwidth; on one GPU the
NVLink leg cannot be measured, so this bounds the kernel's own data-movement efficiency.

  python tools/a2a_bench.py [--P 8] [--seq 32768] [--hq 32] [--hkv 8] [--d 64]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2604_27089_b200 import _lib, kernels

ap = argparse.ArgumentParser()
ap.add_argument("--P", type=int, default=8)
ap.add_argument("--seq", type=int, default=32768)
ap.add_argument("--hq", type=int, default=32)
ap.add_argument("--hkv", type=int, default=8)
ap.add_argument("--d", type=int, default=64)
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--graph", action="store_true",
                help="capture one round in a CUDA graph and replay it: GPU time without the "
                     "host-side launch gaps (epochs are frozen at capture, so the flag waits "
                     "pass immediately on replays; the data movement is real)")
a = ap.parse_args()
P, S, hq, hkv, d = a.P, a.seq, a.hq, a.hkv, a.d
sl = S // P
dev = "cuda"
# source: each rank's packed QKV projection output [1, s/P, (hq+2hkv)*d] (read in place)
srcs = [torch.randn(1, sl, (hq + 2 * hkv) * d, device=dev).bfloat16() for _ in range(P)]
qn, kn = (hq // P) * S * d, (hkv // P) * S * d
regions = [torch.empty(qn + 2 * kn, dtype=torch.bfloat16, device=dev) for _ in range(P)]
flags = torch.zeros((P, _lib.FLAG_WORDS), dtype=torch.int32, device=dev)
fptr = [flags[j].data_ptr() for j in range(P)]
rptr = [x.data_ptr() for x in regions]
epoch = [0]


def call_rank(r, e):
    v = srcs[r].view(1, sl, hq + 2 * hkv, d)
    descs = [kernels.a2a_tensor_desc(v[:, :, :hq], hq, 0, ((hq // P) * S * d, d, S * d)),
             kernels.a2a_tensor_desc(v[:, :, hq:hq + hkv], hkv, qn * 2,
                                     ((hkv // P) * S * d, d, S * d)),
             kernels.a2a_tensor_desc(v[:, :, hq + hkv:], hkv, (qn + kn) * 2,
                                     ((hkv // P) * S * d, d, S * d))]
    return kernels.a2a_launch(_lib.SEQ_TO_HEAD, descs, 1, S, d, 2, P, r, rptr, fptr, e)


def one_round():
    epoch[0] += 1
    e = epoch[0]
    kernels.a2a_mark_ready(fptr, e)  # loopback: all virtual ranks reached epoch e
    for r in range(P):
        chk = call_rank(r, e)
    for r in range(P):
        kernels.a2a_wait(fptr[r], P, r, e, chk)


for _ in range(3):
    one_round()
torch.cuda.synchronize()
run = one_round
if a.graph:
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(side):
        with torch.cuda.graph(graph, stream=side):
            one_round()
    torch.cuda.synchronize()
    run = graph.replay
    for _ in range(3):
        run()
    torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.iters):
    run()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.iters
per_rank = sl * (hq + 2 * hkv) * d * 2  # bytes each rank sends (incl. its own slab)
moved = P * per_rank * 2                # read + write, all virtual ranks, per round
try:
    peak = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
except Exception:
    peak = 6650.0
gbs = moved / (ms / 1e3) / 1e9
print(json.dumps({"kernel": "a2a_push (seq->head, q/k/v in one launch) x P virtual ranks",
                  "timing": "CUDA graph replay (GPU time)" if a.graph else "eager launches",
                  "P": P, "seq": S, "hq": hq, "hkv": hkv, "d": d,
                  "ms_per_round_all_ranks": ms, "ms_per_rank_call": ms / P,
                  "bytes_sent_per_rank": per_rank,
                  "hbm_gbs_read_plus_write": gbs, "hbm_peak_gbs": peak,
                  "frac_of_hbm_copy": gbs / peak,
                  "nvlink_time_model_ms": per_rank * (P - 1) / P / 770e9 * 1e3}))
