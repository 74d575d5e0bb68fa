"""Pin the CPU oracle (oracle/seqcomp_oracle.py) to the reference's own outputs.

The fixtures in tests/golden/ were produced by running the reference
simulator itself (tests/golden/make_golden.py).  When /root/reference is
present (this container, not the GPU box) a few tests additionally compare
against the live reference on fresh seeds."""

import numpy as np
import pytest

from conftest import reference_available
from oracle import seqcomp_oracle as orc


def test_a2a_matches_reference_fixture(golden_dir):
    z = np.load(golden_dir / "a2a.npz")
    for P in (2, 4, 8):
        full = z[f"P{P}_full"]
        sl = full.shape[1] // P
        shards = [full[:, r * sl:(r + 1) * sl] for r in range(P)]
        s2h = orc.all_to_all_shards("seq_to_head", shards)
        assert all(a.dtype == np.uint16 for a in s2h)
        np.testing.assert_array_equal(np.stack(s2h), z[f"P{P}_s2h"])
        h2s = orc.all_to_all_shards("head_to_seq", s2h)
        np.testing.assert_array_equal(np.stack(h2s), z[f"P{P}_h2s"])
        for a, b in zip(h2s, shards):  # round trip (ref tests/test_executor.py:22-29)
            np.testing.assert_array_equal(a, b)


def test_a2a_rejects_bad_direction_and_shapes():
    x = np.zeros((1, 2, 2, 1))
    with pytest.raises(orc.OracleError):
        orc.all_to_all_shards("sideways", [x, x])
    with pytest.raises(orc.OracleError):
        orc.all_to_all_shards("seq_to_head", [x, np.zeros((1, 2, 4, 1))])


def test_attention_matches_reference_fixture(golden_dir):
    z = np.load(golden_dir / "attention.npz")
    for i in range(3):
        x = z[f"c{i}_x"]
        o, lse = orc.attention_fwd(x, x, x)
        assert orc.max_rel_err(o, z[f"c{i}_out"]) <= 1e-12
        assert np.all(np.isfinite(lse))


def _fd_check(q, k, v, seed=0, eps=1e-6):
    rng = np.random.default_rng(seed)
    do = rng.standard_normal(q.shape)
    dq, dk, dv = orc.attention_bwd(q, k, v, do)
    worst = 0.0
    for t, g in ((q, dq), (k, dk), (v, dv)):
        for _ in range(12):
            idx = tuple(int(rng.integers(0, n)) for n in t.shape)
            tp, tm = t.copy(), t.copy()
            tp[idx] += eps
            tm[idx] -= eps
            args_p = [tp if a is t else a for a in (q, k, v)]
            args_m = [tm if a is t else a for a in (q, k, v)]
            fp = np.sum(orc.attention_fwd(*args_p)[0] * do)
            fm = np.sum(orc.attention_fwd(*args_m)[0] * do)
            num = (fp - fm) / (2 * eps)
            worst = max(worst, abs(num - g[idx]) / max(abs(num), abs(g[idx]), 1e-8))
    return worst


@pytest.mark.parametrize("hq,hkv", [(2, 2), (4, 2), (4, 1)])
def test_attention_bwd_finite_differences(hq, hkv):
    rng = np.random.default_rng(hq * 10 + hkv)
    b, s, d = 1, 12, 8
    q = rng.standard_normal((b, s, hq, d))
    k = rng.standard_normal((b, s, hkv, d))
    v = rng.standard_normal((b, s, hkv, d))
    assert _fd_check(q, k, v) < 1e-6


def test_lse_is_logsumexp():
    rng = np.random.default_rng(3)
    q = rng.standard_normal((1, 9, 2, 4))
    _, lse = orc.attention_fwd(q, q, q)
    sc = np.einsum("bqhd,bkhd->bhqk", q, q) / 2.0
    sc = sc + orc.causal_mask(9)
    np.testing.assert_allclose(lse, np.log(np.exp(sc).sum(-1)), rtol=1e-12)


def _check_model(golden_dir, name, tol):
    z = np.load(golden_dir / f"model_{name}.npz")
    b, s, h, d, f, L, P, seed, prec = (int(v) for v in z["dims"])
    dims = orc.Dims(b=b, s=s, h=h, d=d, d_ffn=f, layers=L)
    ids, params = orc.random_leaves(dims, seed)
    names = orc.param_names(dims)
    np.testing.assert_allclose([params[n].sum() for n in names], z["param_checksums"],
                               rtol=1e-12)
    res = orc.sp_forward_backward(dims, ids, params, P)
    assert orc.max_rel_err(np.array(res.loss), z["loss_per_rank"]) <= tol
    tg = res.total_grads()
    if "hidden" in z:
        assert orc.max_rel_err(res.full_hidden(), z["hidden"]) <= tol
        for i, n in enumerate(names):
            assert orc.max_rel_err(tg[n], z[f"grad_{i}"]) <= tol, n
    else:
        rows = z["hidden_rows"]
        assert orc.max_rel_err(res.full_hidden()[:, rows], z["hidden_sample"]) <= tol
        for i, n in enumerate(names):
            flat = tg[n].reshape(-1)
            assert orc.max_rel_err(flat[z[f"grad_{i}_idx"]], z[f"grad_{i}_val"]) <= tol, n
            assert abs(np.linalg.norm(flat) / z[f"grad_{i}_norm"] - 1) <= tol


@pytest.mark.parametrize("name", ["tiny_p2", "tiny_p4"])
def test_model_matches_reference_fixture_full(golden_dir, name):
    _check_model(golden_dir, name, 1e-10)


@pytest.mark.parametrize("name", ["c1_p2", "c1_p1"])
def test_model_c1_matches_reference_fixture_sampled(golden_dir, name):
    # the reference's own SP-equivalence tolerance is 1e-12 (test_acceptance.py:98);
    # elementwise max_rel_err over sampled gradient coordinates near zero needs a
    # looser floor, so pin at 1e-8.
    _check_model(golden_dir, name, 1e-8)


def test_sp_equivalence_property():
    dims = orc.Dims(b=1, s=16, h=4, d=4, d_ffn=8, layers=2)
    ids, params = orc.random_leaves(dims, 5)
    r1 = orc.sp_forward_backward(dims, ids, params, 1)
    r4 = orc.sp_forward_backward(dims, ids, params, 4)
    assert orc.max_rel_err(r1.full_hidden(), r4.full_hidden()) <= 1e-12
    g1, g4 = r1.total_grads(), r4.total_grads()
    for k in g1:
        assert orc.max_rel_err(g1[k], g4[k]) <= 1e-10


@pytest.mark.skipif(not reference_available(), reason="reference not mounted")
@pytest.mark.parametrize("seed", range(3))
def test_oracle_vs_live_reference_random_configs(seed):
    import sys
    sys.path.insert(0, "/root/reference/pkg/src")
    from seqcomp.executor import all_to_all_shards, _eval_attention_core, _causal_mask
    rng = np.random.default_rng(seed)
    P = int(rng.choice([2, 4]))
    shards = [rng.standard_normal((1, 4, 8, 3)) for _ in range(P)]
    for dirn in ("seq_to_head", "head_to_seq"):
        a = all_to_all_shards(dirn, shards)
        b = orc.all_to_all_shards(dirn, shards)
        for x, y in zip(a, b):
            np.testing.assert_array_equal(x, y)
    x = rng.standard_normal((2, 20, 3, 5))
    assert orc.max_rel_err(orc.attention_fwd(x, x, x)[0],
                           _eval_attention_core(x, _causal_mask(20, np.float64))) <= 1e-12
