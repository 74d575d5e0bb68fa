"""bench.py's N > 1 path end to end: torchrun with 2 ranks sharing the one GPU (gloo for
the torch.distributed plumbing via AUTOSP_BENCH_BACKEND; the reshards still go through
the IPC-mapped push kernels), Ulysses SP over the 2 ranks and ZeRO-1.  Checks the one
JSON line rank 0 prints (the numbers are not scaling data: the ranks share a GPU)."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def test_bench_two_ranks_one_gpu():
    env = dict(os.environ, AUTOSP_BENCH_BACKEND="gloo", CUDA_MODULE_LOADING="EAGER")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29531", str(ROOT / "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "3", "--layers", "2", "--seq", "8192",
           "--zero1", "on"]  # (auto would replicate this small model's optimizer state)
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["gpu_launches"] > 0
    assert d["config"]["parallelism"] == "sp2+zero1"
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
    assert d["final_loss"] == d["final_loss"]  # finite (not NaN)
    # all-to-all block: bytes per call (algorithmic, (P-1)/P of the local share), time, GB/s
    # of the standalone reshard launches -- one per layer (dO + delta in the backward); the
    # q/k/v, O and gradient reshards run inside K0 / K3 / K4's epilogues
    a = d["a2a"]
    assert a["calls_per_step"] >= 2 and a["bytes_per_call"] > 0 and a["gbs"] > 0
    assert 0 < a["frac"] and a["peak_gbs"] == 900.0
    # sp_ac block: the seq-aware plan really ran (recomputation) next to save-all
    sp = d["sp_ac"]
    assert sp["mode"] == "seq-aware" and sp["recomputed_fw_nodes"] > 0
    assert sp["step_time_ratio"] > 0 and sp["peak_mem_ratio"] > 0
