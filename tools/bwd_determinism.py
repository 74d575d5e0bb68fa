"""Run-to-run determinism of the attention backward (K4): the same inputs twice, dq/dk/dv
compared bit for bit, for the plain and GQA-split kernels (AUTOSP_BWD_HSPLIT is read once
per process, so each mode runs in its own process).

usage: python tools/bwd_determinism.py [hq hkv s d]"""

import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def one(hq, hkv, s, d, reps=5):
    import torch
    from paper_2604_27089_b200 import kernels
    g = torch.Generator(device="cuda").manual_seed(0)
    q = torch.randn(1, hq, s, d, device="cuda", generator=g).bfloat16()
    k = torch.randn(1, hkv, s, d, device="cuda", generator=g).bfloat16()
    v = torch.randn(1, hkv, s, d, device="cuda", generator=g).bfloat16()
    do = torch.randn(1, hq, s, d, device="cuda", generator=g).bfloat16()
    o, lse = kernels.attn_fwd(q, k, v)
    ref = kernels.attn_bwd(q, k, v, o, do, lse)
    diff = {"dq": 0, "dk": 0, "dv": 0}
    for _ in range(reps):
        got = kernels.attn_bwd(q, k, v, o, do, lse)
        for n, a, b in zip(("dq", "dk", "dv"), got, ref):
            diff[n] += int((a.view(torch.int16) != b.view(torch.int16)).sum())
    torch.cuda.synchronize()
    print(f"hsplit={os.environ.get('AUTOSP_BWD_HSPLIT', '0')} hq={hq} hkv={hkv} s={s} d={d}: "
          f"elements differing over {reps} reruns: {diff}", flush=True)


if __name__ == "__main__":
    if os.environ.get("_BWD_DET_CHILD"):
        one(*map(int, sys.argv[1:5]))
    else:
        shape = sys.argv[1:5] or ["8", "4", "4096", "64"]
        for mode in ("1", "2"):
            env = dict(os.environ, AUTOSP_BWD_HSPLIT=mode, _BWD_DET_CHILD="1")
            subprocess.run([sys.executable, __file__, *shape], env=env, check=True)
