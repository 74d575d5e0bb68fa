"""Trainability planner (planner.py): calibrated against the measured single-GPU
frontier of the Llama-3-8B shape (192K fits, 224K OOMs on one B200) and monotone in P."""

from paper_2604_27089_b200.planner import predict_max_context, step_memory
from paper_2604_27089_b200.workloads import CONFIGS

DEV = 178.35 * 2 ** 30


def test_single_gpu_frontier_matches_measurement():
    cfg = CONFIGS["llama3-8b"]
    s = predict_max_context(cfg, 1, DEV)
    assert 163840 <= s <= 229376  # measured: 196608 trains, 229376 runs out of memory
    assert step_memory(cfg, 229376, 1).total > 0.97 * DEV


def test_more_ranks_never_shorter():
    for name in ("llama3-8b", "llama3.2-1b"):
        cfg = CONFIGS[name]
        prev = 0
        for P in (1, 2, 4, 8):
            s = predict_max_context(cfg, P, DEV)
            assert s >= prev and s % (16 * 128 * P) == 0
            prev = s
