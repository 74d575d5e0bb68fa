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


def test_symmetric_heap_term_matches_the_op_slabs():
    """at P > 1 the planner models the symmetric receive heap (which
    now grows on demand) with the exact slab sizes ops.py allocates: per layer one q/k/v
    slab + one token-major O slab kept, plus one layer's backward reshards."""
    from paper_2604_27089_b200.planner import pool_bytes, pool_layer_bytes
    cfg = CONFIGS["llama3-8b"]
    S, P = 524288, 8
    kept, bwd = pool_layer_bytes(cfg, S, P)
    sl, hd = S // P, cfg.head_dim
    assert kept == 2 * S * (cfg.hq + 2 * cfg.hkv) // P * hd + 2 * sl * cfg.hq * hd
    assert pool_bytes(cfg, S, P) == cfg.layers * kept + bwd
    assert abs(pool_bytes(cfg, S, P) / 1e9 - 43.5) < 1.0      # ~43 GB per rank at 512K
    est = step_memory(cfg, S, P)
    assert est.pool == pool_bytes(cfg, S, P)
    assert est.total == est.static + est.saved + est.pool + est.transient
    assert est.total < 0.97 * DEV                             # C4 512K at SP=8 fits
    assert step_memory(cfg, S, 1).pool == 0
