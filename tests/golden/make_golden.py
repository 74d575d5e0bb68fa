"""Generate the golden fixtures under tests/golden/ by running the REFERENCE
simulator (``seqcomp``, read-only at /root/reference/pkg/src) in this
container.  The fixtures pin ``oracle/seqcomp_oracle.py`` (and through it the
CUDA path) to the reference's own outputs; /root/reference does not exist on
the GPU box, so only these committed .npz files travel.

Run:  python tests/golden/make_golden.py   (needs /root/reference)

Reference entry points used (file:line under /root/reference/pkg/src/seqcomp):
  all_to_all_shards      executor.py:203-230
  _eval_attention_core   executor.py:132-142
  build_transformer_graph transformer.py:42-113, transform_sp sp_pass.py:133-220,
  lower lowering.py:42, build_joint_graph autodiff.py:266, execute_ranks executor.py:344
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


def _ref():
    sys.path.insert(0, str(REF))
    import seqcomp.executor as ex
    from seqcomp.autodiff import build_joint_graph
    from seqcomp.ir import OpKind
    from seqcomp.lowering import lower
    from seqcomp.sp_pass import SPConfig, transform_sp
    from seqcomp.transformer import ModelDims, build_transformer_graph
    return ex, build_joint_graph, OpKind, lower, SPConfig, transform_sp, ModelDims, \
        build_transformer_graph


def _leaves(g, rng, OpKind, scale=0.1):
    # same procedure as the reference's tests/helpers.py:21-28
    inputs, params = {}, {}
    for n in g.nodes:
        if n.kind is OpKind.INPUT:
            inputs[n.id] = rng.integers(0, 64, size=n.out.extents()).astype(np.float64)
        elif n.kind is OpKind.PARAMETER:
            params[n.id] = rng.standard_normal(n.out.extents()) * scale
    return inputs, params


def model_fixture(name, b, s, h, d, d_ffn, layers, P, seed, full, precision=64):
    ex, build_joint_graph, OpKind, lower, SPConfig, transform_sp, ModelDims, build = _ref()
    dims = ModelDims(b=b, s=s, h=h, d=d, d_ffn=d_ffn, layers=layers)
    g = build(dims)
    spg = transform_sp(g, SPConfig(world_size=P))
    sp_low = lower(spg.graph)
    j = build_joint_graph(sp_low)
    rng = np.random.default_rng(seed)
    # draw leaves on the unsharded graph, re-key by position (test_acceptance.py:77-84)
    low = lower(g)
    full_in, full_par = _leaves(low, rng, OpKind)
    def rekey(arrs, kind):
        a = [n.id for n in low.nodes if n.kind is kind]
        bb = [n.id for n in sp_low.nodes if n.kind is kind]
        return {y: arrs[x] for x, y in zip(a, bb)}
    inputs, params = rekey(full_in, OpKind.INPUT), rekey(full_par, OpKind.PARAMETER)
    outs = ex.execute_ranks(j.graph, ex.DeviceGroup(P=P), inputs, params, precision=precision)
    hidden = np.concatenate([o[j.graph.outputs[0]] for o in outs], axis=1)
    loss = np.array([float(o[j.graph.outputs[1]]) for o in outs])
    pids = [n.id for n in sp_low.nodes if n.kind is OpKind.PARAMETER]
    grads = [sum(o[j.grad_map[p]] for o in outs) for p in pids]
    pvals = [params[p] for p in pids]
    rec = {"dims": np.array([b, s, h, d, d_ffn, layers, P, seed, precision]),
           "loss_per_rank": loss,
           "param_checksums": np.array([float(np.sum(v)) for v in pvals])}
    if full:
        rec["hidden"] = hidden
        for i, gv in enumerate(grads):
            rec[f"grad_{i}"] = gv
    else:
        srng = np.random.default_rng(1000 + seed)
        rec["hidden_rows"] = srng.choice(hidden.shape[1], size=16, replace=False)
        rec["hidden_sample"] = hidden[:, rec["hidden_rows"]]
        for i, gv in enumerate(grads):
            flat = gv.reshape(-1)
            idx = srng.choice(flat.size, size=min(256, flat.size), replace=False)
            rec[f"grad_{i}_idx"] = idx
            rec[f"grad_{i}_val"] = flat[idx]
            rec[f"grad_{i}_norm"] = np.array(np.linalg.norm(flat))
    np.savez_compressed(OUT / f"model_{name}.npz", **rec)
    print(f"model_{name}: loss={loss.sum():.6e}")


def a2a_fixture():
    ex = _ref()[0]
    rec = {}
    for P, (b, s, h, d) in {2: (1, 8, 4, 8), 4: (2, 16, 8, 8), 8: (1, 64, 8, 16)}.items():
        rng = np.random.default_rng(P)
        full = rng.integers(0, 1 << 16, size=(b, s, h, d), dtype=np.uint16)  # bf16 bit patterns
        sl = s // P
        shards = [full[:, r * sl:(r + 1) * sl] for r in range(P)]
        s2h = ex.all_to_all_shards("seq_to_head", shards)
        h2s = ex.all_to_all_shards("head_to_seq", s2h)
        rec[f"P{P}_full"] = full
        rec[f"P{P}_s2h"] = np.stack(s2h)
        rec[f"P{P}_h2s"] = np.stack(h2s)
    np.savez_compressed(OUT / "a2a.npz", **rec)
    print("a2a fixtures written")


def attention_fixture():
    ex = _ref()[0]
    rec = {}
    for i, (b, s, h, d) in enumerate([(1, 64, 2, 16), (2, 33, 3, 8), (1, 128, 1, 32)]):
        rng = np.random.default_rng(50 + i)
        x = rng.standard_normal((b, s, h, d))
        rec[f"c{i}_x"] = x
        rec[f"c{i}_out"] = ex._eval_attention_core(x, ex._causal_mask(s, np.float64))
    np.savez_compressed(OUT / "attention.npz", **rec)
    print("attention fixtures written")


if __name__ == "__main__":
    a2a_fixture()
    attention_fixture()
    model_fixture("tiny_p2", b=2, s=16, h=4, d=4, d_ffn=16, layers=2, P=2, seed=7, full=True)
    model_fixture("tiny_p4", b=1, s=32, h=4, d=8, d_ffn=16, layers=1, P=4, seed=11, full=True)
    model_fixture("c1_p2", b=1, s=1024, h=8, d=32, d_ffn=1024, layers=2, P=2, seed=0,
                  full=False)
    model_fixture("c1_p1", b=1, s=1024, h=8, d=32, d_ffn=1024, layers=2, P=1, seed=0,
                  full=False)
