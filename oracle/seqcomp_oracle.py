"""CPU oracle for the Ulysses-SP hot path — TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  The CUDA path in
``paper_2604_27089_b200`` never routes through here.

It restates, in NumPy (fp64 by default), the reference simulator
``seqcomp`` (``/root/reference/pkg/src/seqcomp``) for the functions on the
hot path, operation for operation:

* ``all_to_all_shards``      — ``executor.py:203-230`` (pure index permutation)
* ``causal_mask``/``softmax`` — ``executor.py:37-40,62-65``, ``ir.py:19``
* ``attention_fwd``          — ``executor.py:132-142`` / ``lowering.py:82-122``
  extended (beyond the reference, ``SPEC.md:216``) to distinct Q/K/V, GQA
  head groups and a log-sum-exp output
* ``attention_bwd``          — the joint-graph recipes ``autodiff.py:156-162``
  (batch-matmul grads), ``autodiff.py:190-195`` (scale), ``autodiff.py:213-214``
  + ``executor.py:89-91`` (softmax_dx)
* ``rmsnorm*``/``silu*``     — ``executor.py:33-34,43-59,85-88``
* ``SeqcompModel``           — ``transformer.py:42-113`` run under the SP
  rewrite ``sp_pass.py:133-220`` (rank-offset positions ``sp_pass.py:160-163``,
  ``executor.py:68-70``; contiguous sequence shards ``executor.py:324-341``;
  a2a gradient = inverse a2a ``autodiff.py:252-262``).  Loss and parameter
  gradients are per-rank partials that callers sum
  (``tests/test_acceptance.py:87-96``).

Parity pinning: ``tests/golden/make_golden.py`` runs the reference itself
(importable here) and commits its outputs under ``tests/golden/``;
``tests/test_oracle_golden.py`` checks this restatement against them.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

NEG_INF_MASK = -1e9  # ir.py:19
DEFAULT_VOCAB = 64  # transformer.py:17
RMS_EPS = 1e-6  # lowering.py:79, executor.py:158


class OracleError(ValueError):
    """Shape / direction errors (the reference raises CollectiveError / ValidationError)."""


# ---------------------------------------------------------------------------
# all-to-all (executor.py:203-230)
# ---------------------------------------------------------------------------


def all_to_all_shards(direction: str, shards: list[np.ndarray]) -> list[np.ndarray]:
    """Ulysses reshard over axis convention (batch, sequence, heads, head_dim).

    seq_to_head: rank r receives concat_j shard_j[:, :, r*h/P:(r+1)*h/P] along seq.
    head_to_seq: rank r receives concat_j shard_j[:, r*s/P:(r+1)*s/P] along heads.
    Dtype-agnostic (bf16 payloads are passed as uint16 views)."""
    P = len(shards)
    if P == 1:
        return [shards[0].copy()]
    base = shards[0].shape
    if any(x.shape != base for x in shards):
        raise OracleError(f"mismatched shard shapes {[x.shape for x in shards]}")
    if direction == "seq_to_head":
        if base[2] % P:
            raise OracleError(f"heads {base[2]} not divisible by {P}")
        hl = base[2] // P
        return [np.concatenate([x[:, :, r * hl:(r + 1) * hl] for x in shards], axis=1)
                for r in range(P)]
    if direction == "head_to_seq":
        if base[1] % P:
            raise OracleError(f"sequence {base[1]} not divisible by {P}")
        sl = base[1] // P
        return [np.concatenate([x[:, r * sl:(r + 1) * sl] for x in shards], axis=2)
                for r in range(P)]
    raise OracleError(f"unknown all-to-all direction {direction!r}")


def inverse_direction(direction: str) -> str:
    """ir.py:468-469."""
    return "head_to_seq" if direction == "seq_to_head" else "seq_to_head"


# ---------------------------------------------------------------------------
# attention (executor.py:132-142, lowering.py:82-122, autodiff.py recipes)
# ---------------------------------------------------------------------------


def causal_mask(s: int, dtype=np.float64) -> np.ndarray:
    m = np.zeros((s, s), dtype=dtype)
    m[np.triu_indices(s, k=1)] = NEG_INF_MASK
    return m


def softmax(x: np.ndarray) -> np.ndarray:
    m = np.max(x, axis=-1, keepdims=True)
    e = np.exp(x - m)
    return e / np.sum(e, axis=-1, keepdims=True)


def _expand_kv(k: np.ndarray, hq: int) -> np.ndarray:
    """[b, s, hkv, d] -> [b, s, hq, d]: q head i reads kv head i // (hq/hkv)."""
    hkv = k.shape[2]
    if hq % hkv:
        raise OracleError(f"q heads {hq} not a multiple of kv heads {hkv}")
    return np.repeat(k, hq // hkv, axis=2)


def _probs(q, k, causal, scale):
    qh = np.transpose(q, (0, 2, 1, 3))  # permute [0,2,1,3]
    kt = np.transpose(k, (0, 2, 3, 1))  # permute [0,2,3,1]
    scores = np.matmul(qh, kt)
    scaled = scores * q.dtype.type(scale)
    sq, sk = scaled.shape[-2:]
    if causal:
        scaled = scaled + causal_mask(sq, q.dtype)[:, :sk]
    return scaled, softmax(scaled)


def attention_fwd(q, k, v, causal: bool = True, scale: float | None = None):
    """softmax(q kᵀ/√d + M) v per head.  q [b,s,hq,d], k/v [b,s,hkv,d].

    Returns (o [b,s,hq,d], lse [b,hq,s]) where lse is the natural-log
    log-sum-exp of the masked, scaled scores (what the GPU kernel saves)."""
    hq, d = q.shape[2], q.shape[3]
    scale = 1.0 / math.sqrt(d) if scale is None else scale
    ke, ve = _expand_kv(k, hq), _expand_kv(v, hq)
    scaled, probs = _probs(q, ke, causal, scale)
    ctx = np.matmul(probs, np.transpose(ve, (0, 2, 1, 3)))
    m = np.max(scaled, axis=-1, keepdims=True)
    lse = (m + np.log(np.sum(np.exp(scaled - m), axis=-1, keepdims=True)))[..., 0]
    return np.transpose(ctx, (0, 2, 1, 3)), lse


def attention_bwd(q, k, v, do, causal: bool = True, scale: float | None = None):
    """Gradients of attention_fwd's o w.r.t. q, k, v given do.

    dP = dO Vᵀ; dS = P∘(dP − Σ dP∘P) (softmax_dx); scale; dQ = dS K;
    dK = dSᵀ Q; dV = Pᵀ dO; GQA sums dK/dV over each kv head's q-head group."""
    b, s, hq, d = q.shape
    hkv = k.shape[2]
    scale = 1.0 / math.sqrt(d) if scale is None else scale
    ke, ve = _expand_kv(k, hq), _expand_kv(v, hq)
    _, probs = _probs(q, ke, causal, scale)
    qh = np.transpose(q, (0, 2, 1, 3))
    kh = np.transpose(ke, (0, 2, 1, 3))
    vh = np.transpose(ve, (0, 2, 1, 3))
    doh = np.transpose(do, (0, 2, 1, 3))
    dprobs = np.matmul(doh, np.swapaxes(vh, -1, -2))
    dv = np.matmul(np.swapaxes(probs, -1, -2), doh)
    dmasked = probs * (dprobs - np.sum(dprobs * probs, axis=-1, keepdims=True))
    dscores = dmasked * q.dtype.type(scale)
    dq = np.matmul(dscores, kh)
    dk = np.matmul(np.swapaxes(dscores, -1, -2), qh)
    g, sk = hq // hkv, k.shape[1]  # (sk != s: a query block against a longer key prefix)
    dk = dk.reshape(b, hkv, g, sk, d).sum(axis=2)
    dv = dv.reshape(b, hkv, g, sk, d).sum(axis=2)
    return (np.transpose(dq, (0, 2, 1, 3)), np.transpose(dk, (0, 2, 1, 3)),
            np.transpose(dv, (0, 2, 1, 3)))


# ---------------------------------------------------------------------------
# elementwise recipes (executor.py:33-59, 85-88)
# ---------------------------------------------------------------------------


def silu(x):
    return x / (1.0 + np.exp(-x))


def silu_dx(x, dy):
    sig = 1.0 / (1.0 + np.exp(-x))
    return dy * sig * (1.0 + x * (1.0 - sig))


def rmsnorm(x, w, eps=RMS_EPS):
    r = 1.0 / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps)
    return x * r * w


def rmsnorm_dx(x, w, dy, eps=RMS_EPS):
    n = x.shape[-1]
    ms = np.mean(x * x, axis=-1, keepdims=True) + eps
    r = 1.0 / np.sqrt(ms)
    dyw = dy * w
    return r * dyw - (r / ms / n) * x * np.sum(dyw * x, axis=-1, keepdims=True)


def rmsnorm_dw(x, w, dy, eps=RMS_EPS):
    r = 1.0 / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps)
    return np.sum((dy * x * r).reshape(-1, x.shape[-1]), axis=0)


# ---------------------------------------------------------------------------
# the reference decoder under Ulysses SP (transformer.py:42-113, sp_pass.py)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class Dims:
    """transformer.py:20-39 (ModelDims)."""
    b: int
    s: int
    h: int
    d: int
    d_ffn: int
    layers: int
    vocab: int = DEFAULT_VOCAB

    @property
    def d_model(self) -> int:
        return self.h * self.d


def param_names(dims: Dims) -> list[str]:
    """Parameter creation order of build_transformer_graph (transformer.py:47-104)."""
    names = ["embed_table"]
    for l in range(dims.layers):
        names += [f"l{l}.norm1.w", f"l{l}.qkv.w", f"l{l}.out.w", f"l{l}.norm2.w",
                  f"l{l}.mlp.up.w", f"l{l}.mlp.down.w"]
    return names


def param_shapes(dims: Dims) -> dict[str, tuple[int, ...]]:
    dm, f = dims.d_model, dims.d_ffn
    out = {"embed_table": (dims.vocab, dm)}
    for l in range(dims.layers):
        out.update({f"l{l}.norm1.w": (dm,), f"l{l}.qkv.w": (dm, dm), f"l{l}.out.w": (dm, dm),
                    f"l{l}.norm2.w": (dm,), f"l{l}.mlp.up.w": (f, dm),
                    f"l{l}.mlp.down.w": (dm, f)})
    return out


def random_leaves(dims: Dims, seed: int, scale: float = 0.1):
    """Same draw order/distribution as the reference fixtures
    (``tests/helpers.py:21-28``): token ids first, then N(0, scale²)
    parameters in graph creation order."""
    rng = np.random.default_rng(seed)
    ids = rng.integers(0, 64, size=(dims.b, dims.s)).astype(np.float64)
    shapes = param_shapes(dims)
    params = {n: rng.standard_normal(shapes[n]) * scale for n in param_names(dims)}
    return ids, params


@dataclass
class SPResult:
    hidden: list[np.ndarray]  # per-rank [b, s/P, d_model]
    loss: list[float]  # per-rank partial losses
    grads: list[dict[str, np.ndarray]] = field(default_factory=list)  # per-rank partials

    def full_hidden(self) -> np.ndarray:
        return np.concatenate(self.hidden, axis=1)

    def total_loss(self) -> float:
        return float(sum(self.loss))

    def total_grads(self) -> dict[str, np.ndarray]:
        return {k: sum(g[k] for g in self.grads) for k in self.grads[0]}


def _linear(x, w):  # executor.py:155-156
    return np.matmul(x, w.T)


def sp_forward_backward(dims: Dims, ids: np.ndarray, params: dict, P: int,
                        backward: bool = True, dtype=np.float64) -> SPResult:
    """Run the reference decoder on P lockstep ranks (Ulysses layout toggle
    around every attention), returning per-rank hidden/loss/grad partials."""
    b, s, h, d = dims.b, dims.s, dims.h, dims.d
    if s % P or h % P:
        raise OracleError(f"s={s}, h={h} not divisible by P={P}")
    sl = s // P
    prm = {k: np.asarray(v, dtype=dtype) for k, v in params.items()}
    ids_r = [np.asarray(ids)[:, r * sl:(r + 1) * sl] for r in range(P)]
    table = prm["embed_table"]
    x = []
    for r in range(P):
        emb = table[ids_r[r].astype(np.int64) % table.shape[0]]
        pos = np.arange(r * sl, (r + 1) * sl, dtype=dtype).reshape(sl, 1)
        x.append(emb + pos)
    caches = []
    for l in range(dims.layers):
        c = {"x_in": x}
        n1 = [rmsnorm(xi, prm[f"l{l}.norm1.w"]) for xi in x]
        qkv = [_linear(ni, prm[f"l{l}.qkv.w"]).reshape(b, sl, h, d) for ni in n1]
        xh = all_to_all_shards("seq_to_head", qkv) if P > 1 else qkv
        att = [attention_fwd(t, t, t)[0] for t in xh]
        ao = all_to_all_shards("head_to_seq", att) if P > 1 else att
        ao = [a.reshape(b, sl, h * d) for a in ao]
        x_mid = [_linear(a, prm[f"l{l}.out.w"]) + xi for a, xi in zip(ao, x)]
        n2 = [rmsnorm(xm, prm[f"l{l}.norm2.w"]) for xm in x_mid]
        up = [_linear(ni, prm[f"l{l}.mlp.up.w"]) for ni in n2]
        act = [silu(u) for u in up]
        x = [_linear(a, prm[f"l{l}.mlp.down.w"]) + xm for a, xm in zip(act, x_mid)]
        c.update(n1=n1, xh=xh, ao=ao, x_mid=x_mid, n2=n2, up=up, act=act)
        caches.append(c)
    res = SPResult(hidden=x, loss=[float(np.sum(xi * xi)) for xi in x])
    if not backward:
        return res

    grads = [{k: np.zeros_like(v) for k, v in prm.items()} for _ in range(P)]
    dx = [2.0 * xi for xi in x]  # Loss: square -> mul(dy, x) -> scale 2 (autodiff.py:181-186)
    for l in reversed(range(dims.layers)):
        c = caches[l]
        w = {k: prm[f"l{l}.{k}"] for k in ("norm1.w", "qkv.w", "out.w", "norm2.w",
                                            "mlp.up.w", "mlp.down.w")}
        d_act = []
        for r in range(P):
            g = grads[r]
            g[f"l{l}.mlp.down.w"] += dx[r].reshape(-1, dx[r].shape[-1]).T @ \
                c["act"][r].reshape(-1, c["act"][r].shape[-1])
            d_act.append(dx[r] @ w["mlp.down.w"])
        d_n2 = []
        for r in range(P):
            d_up = silu_dx(c["up"][r], d_act[r])
            grads[r][f"l{l}.mlp.up.w"] += d_up.reshape(-1, d_up.shape[-1]).T @ \
                c["n2"][r].reshape(-1, c["n2"][r].shape[-1])
            d_n2.append(d_up @ w["mlp.up.w"])
        d_mid = []
        for r in range(P):
            grads[r][f"l{l}.norm2.w"] += rmsnorm_dw(c["x_mid"][r], w["norm2.w"], d_n2[r])
            d_mid.append(rmsnorm_dx(c["x_mid"][r], w["norm2.w"], d_n2[r]) + dx[r])
        d_ao = []
        for r in range(P):
            grads[r][f"l{l}.out.w"] += d_mid[r].reshape(-1, d_mid[r].shape[-1]).T @ \
                c["ao"][r].reshape(-1, c["ao"][r].shape[-1])
            d_ao.append((d_mid[r] @ w["out.w"]).reshape(b, sl, h, d))
        # grad of a2a(head_to_seq) = a2a(seq_to_head)  (autodiff.py:252-262)
        d_att = all_to_all_shards("seq_to_head", d_ao) if P > 1 else d_ao
        d_xh = []
        for r in range(P):
            t = c["xh"][r]
            dq, dk, dv = attention_bwd(t, t, t, d_att[r])
            d_xh.append(dq + dk + dv)  # q = k = v share one value
        d_qkv = all_to_all_shards("head_to_seq", d_xh) if P > 1 else d_xh
        new_dx = []
        for r in range(P):
            dqkv = d_qkv[r].reshape(b, sl, h * d)
            grads[r][f"l{l}.qkv.w"] += dqkv.reshape(-1, h * d).T @ \
                c["n1"][r].reshape(-1, h * d)
            d_n1 = dqkv @ w["qkv.w"]
            grads[r][f"l{l}.norm1.w"] += rmsnorm_dw(c["x_in"][r], w["norm1.w"], d_n1)
            new_dx.append(rmsnorm_dx(c["x_in"][r], w["norm1.w"], d_n1) + d_mid[r])
        dx = new_dx
    for r in range(P):  # scatter_add_rows (executor.py:120-128)
        idx = ids_r[r].astype(np.int64).reshape(-1) % table.shape[0]
        np.add.at(grads[r]["embed_table"], idx, dx[r].reshape(-1, dx[r].shape[-1]))
    res.grads = grads
    return res


# ---------------------------------------------------------------------------
# comparison metrics (norm-aware, plus the reference's max_rel_err)
# ---------------------------------------------------------------------------


def max_rel_err(a, b) -> float:
    """executor.py:466-470 (elementwise, 1e-12 floor)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.maximum(np.maximum(np.abs(a), np.abs(b)), 1e-12)
    return float(np.max(np.abs(a - b) / den))


def norm_rel_err(a, ref) -> float:
    """max|a − ref| / max|ref| — the bf16 parity metric."""
    a = np.asarray(a, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    den = max(float(np.max(np.abs(ref))), 1e-30)
    return float(np.max(np.abs(a - ref))) / den
