"""``sp_ac`` — sequence-aware activation checkpointing as an AOTAutograd partitioner.

Reference: ``ac_pass.py`` (``AcMode`` :26-29, ``guarded_nodes`` :103-114,
``build_flow_network`` :117-139, ``min_cut`` :142-178).  The joint forward+backward
graph is turned into a split-node flow network — node ``n`` becomes ``n_in -> n_out``
with capacity = bytes of its output, data edges and source/sink wiring are infinite —
and the minimum source/sink cut picks the cheapest set of forward values to keep; every
other value the backward needs is recomputed in the backward graph.

Modes differ only in which forward nodes get an infinite source edge (a *guard*: may
not be recomputed):

* ``conservative``  every matmul + the AutoSP ops  (≈ torch's default policy)
* ``seq-aware``     only the attention region (default; the paper's sp_ac): projections
                    and MLP matmuls may be recomputed, attention never is
* ``seq-aware-all`` no matmul guards

Deliberate divergence from the reference (SURVEY §0 findings 2/3, north star): in every
mode the all-to-all outputs and the attention outputs (O, LSE) are guarded, so backward
never re-issues communication and never re-runs the O(s^2) forward; the saved state of
attention is O + LSE (flash-style), never the probabilities.
"""

from __future__ import annotations

import operator
from enum import Enum

import torch
import torch.fx as fx

from .errors import InfeasibleError


class AcMode(str, Enum):  # ac_pass.py:26-29
    CONSERVATIVE = "conservative"
    SEQ_AWARE_NON_ATTENTION = "seq-aware"
    SEQ_AWARE_ALL = "seq-aware-all"
    # trainability planner (the paper enables SAC only when the
    # un-checkpointed step would not fit): keep every activation the
    # backward needs if that fits the device budget, else fall back to seq-aware.
    AUTO = "auto"


MEMORY_FRACTION = 0.90   # of total device memory usable by one step
STATE_MULTIPLIER = 4     # params + grads + 2 optimizer moments, in the parameter dtype
TRANSIENT_MARGIN = 1.25  # backward working set on top of the saved activations


RECOMPUTE_PENALTY = 0.05  # fraction of a node's bytes charged when it is recomputed
MATMUL_PENALTY = 4.0      # matmuls cost more to recompute than elementwise ops
_MATMULS = {"mm", "addmm", "bmm", "baddbmm", "matmul", "linear", "_scaled_mm"}


def _opname(n: fx.Node) -> str:
    t = n.target
    if hasattr(t, "_schema"):
        return t._schema.name  # e.g. "aten::mm", "autosp::all_to_all"
    return getattr(t, "__name__", str(t))


def is_autosp_collective(n: fx.Node) -> bool:
    return n.op == "call_function" and _opname(n) in ("autosp::all_to_all",
                                                      "autosp::attention_a2a",
                                                      "autosp::ulysses_qkv_attention",
                                                      "autosp::ulysses_qkv_proj_attention",
                                                      "autosp::qkv_grad_gather",
                                                      "autosp::qkv_attention_grad",
                                                      "autosp::grad_out_reshard")


def is_autosp_attention(n: fx.Node) -> bool:
    return n.op == "call_function" and _opname(n) in ("autosp::attention",
                                                      "autosp::attention_a2a",
                                                      "autosp::ulysses_qkv_attention",
                                                      "autosp::ulysses_qkv_proj_attention")


def _is_matmul(n: fx.Node) -> bool:
    name = _opname(n)
    return name.startswith("aten::") and name[6:] in _MATMULS


_VIEWS = {"aten::t", "aten::view", "aten::_unsafe_view", "aten::transpose", "aten::permute",
          "aten::expand", "aten::slice", "aten::alias", "aten::detach", "aten::reshape",
          "aten::unsqueeze", "aten::squeeze"}


def _aliases_input(n: fx.Node) -> bool:
    """A graph input (parameter / user input) or a view of one: alive anyway during the
    backward, so keeping it costs no memory (a pure byte min-cut would charge the weight
    transposes every layer's matmul backward needs)."""
    while n.op == "call_function" and _opname(n) in _VIEWS and n.args and \
            isinstance(n.args[0], fx.Node):
        n = n.args[0]
    return n.op == "placeholder"


def _nbytes(n: fx.Node) -> int | None:
    v = n.meta.get("val")
    if isinstance(v, torch.Tensor):
        return v.numel() * v.element_size()
    if isinstance(v, (int, float, bool, torch.SymInt)) or v is None:
        return 0 if not isinstance(v, torch.Tensor) and n.op == "placeholder" else None
    return None  # tuples / lists: cannot be saved as a unit


_NORMS = {"aten::_fused_rms_norm", "aten::rms_norm", "aten::native_layer_norm",
          "autosp::rms_norm"}
_CASTS = {"aten::_to_copy", "prims::convert_element_type"}


def _norm_input(n: fx.Node) -> bool:
    """n enters a normalisation: a fused norm op, or a decomposed RMSNorm
    ``x * rsqrt(mean(x^2) + eps)`` (possibly after an fp32 cast of x)."""
    for u in n.users:
        if u.op != "call_function":
            continue
        name = _opname(u)
        if name in _NORMS and u.args and u.args[0] is n:
            return True
        if name in _CASTS and _norm_input_decomposed(u):
            return True
    return _norm_input_decomposed(n)


def _norm_input_decomposed(n: fx.Node) -> bool:
    users = [u for u in n.users if u.op == "call_function"]
    has_sq = any(_opname(u) == "aten::pow" for u in users)
    has_scale = any(_opname(u) == "aten::mul" and any(
        isinstance(a, fx.Node) and _opname(a) == "aten::rsqrt" for a in u.args) for u in users)
    return has_sq and has_scale


def is_residual_boundary(n: fx.Node) -> bool:
    """Values entering a normalisation = the residual stream (x_in before attention,
    x_mid before the MLP, the final hidden state)."""
    return n.op == "call_function" and _norm_input(n)


def is_layer_boundary(n: fx.Node, fw: set | None = None, max_nodes: int = 512) -> bool:
    """The residual value entering a layer's pre-attention norm (x_in).  Guarding these
    gives per-layer checkpoints: everything from x_in to the next x_in except attention
    and the a2a outputs (norms, projections, RoPE, the mid-layer residual x_mid, the MLP)
    is recomputable; the min-cut cannot "recompute" a residual value through the whole
    network (0 bytes in a pure byte min-cut but O(L^2) time).  x_in is recognised by
    reaching an attention / all-to-all through exactly one projection matmul without
    crossing another residual value (searching forward nodes only when the joint graph's
    forward set ``fw`` is given: backward nodes reach everything)."""
    if not is_residual_boundary(n):
        return False
    seen = {n}
    frontier = [(u, 0) for u in n.users]
    while frontier and len(seen) < max_nodes:
        u, mm = frontier.pop()
        if u in seen or u.op != "call_function" or (fw is not None and u not in fw):
            continue
        seen.add(u)
        if is_autosp_attention(u) or is_autosp_collective(u):
            return True
        if is_residual_boundary(u):
            continue
        k = mm + (1 if _is_matmul(u) else 0)
        if k > 1:
            continue
        frontier.extend((w, k) for w in u.users)
    return False


def is_random(n: fx.Node) -> bool:
    """Ops drawing random numbers (dropout, rand*, bernoulli, ...): a recomputation in the
    backward would draw a DIFFERENT mask than the forward used (torch's own min-cut
    partitioner bans them from recomputation for the same reason)."""
    if n.op != "call_function":
        return False
    tags = getattr(n.target, "tags", ())
    return torch.Tag.nondeterministic_seeded in tags


def guarded(n: fx.Node, mode: AcMode, fw: set | None = None) -> bool:
    """Forward nodes that must not be recomputed (ac_pass.py:103-114 + the AutoSP guard)."""
    if is_autosp_collective(n) or is_autosp_attention(n) or is_random(n):
        return True
    if is_layer_boundary(n, fw):
        return True
    if n.op == "call_function" and n.target is operator.getitem:
        src = n.args[0]
        if isinstance(src, fx.Node) and (is_autosp_collective(src) or is_autosp_attention(src)):
            return True
    if mode is AcMode.CONSERVATIVE and _is_matmul(n):
        return True
    return False


def plan(joint_module: fx.GraphModule, num_fwd_outputs: int, mode: AcMode):
    """Return (saved_values, saved_sym_nodes, stats) for the joint graph."""
    import networkx as nx
    from torch._functorch.partitioners import classify_nodes

    info = classify_nodes(joint_module, [], num_fwd_outputs)
    # forward side = everything computable without the tangents (values only the backward
    # consumes, e.g. the attention LSE, are still forward values: saved or recomputed)
    fw = {n for n in joint_module.graph.nodes
          if n.op != "output" and n not in info.tangents_closure}
    G = nx.DiGraph()
    INF = float("inf")

    def add(u, v, cap=None):
        if cap is None:
            G.add_edge(u, v)  # no capacity attribute = infinite (networkx)
        else:
            G.add_edge(u, v, capacity=cap)

    for n in joint_module.graph.nodes:
        if n.op == "output":
            continue
        if n in fw:
            if n.op == "placeholder":
                add("source", n.name + "_in")
            b = _nbytes(n)
            sym = isinstance(n.meta.get("val"), torch.SymInt)
            cap = None if (b is None and not sym) else (b or 1)
            if cap is not None and _aliases_input(n):
                cap = 1
            add(n.name + "_in", n.name + "_out", cap)
            if guarded(n, mode, fw):
                add("source", n.name + "_in")
            elif n.op != "placeholder" and b:
                # recompute is not free: a node recomputed in backward (n_in on the sink
                # side) pays a penalty, so long recompute chains lose to saving a small
                # boundary value (the residual stream) -- keeps peak memory bounded
                pen = RECOMPUTE_PENALTY * b * (MATMUL_PENALTY if _is_matmul(n) else 1.0)
                add("source", n.name + "_in", max(1, int(pen)))
            for u in n.users:
                if u in fw:
                    add(n.name + "_out", u.name + "_in")
                elif u.op != "output":
                    add(n.name + "_out", u.name + "_in")
        else:
            add(n.name + "_in", "sink")
            for u in n.users:
                if u.op != "output":
                    add(n.name + "_in", u.name + "_in")
    if "sink" not in G or "source" not in G:
        return [], [], {"cut_bytes": 0}
    try:
        cut_value, (reach, _) = nx.minimum_cut(G, "source", "sink")
    except nx.NetworkXUnbounded:
        inf_only = nx.DiGraph([(u, v) for u, v, d in G.edges(data=True) if "capacity" not in d])
        path = nx.shortest_path(inf_only, "source", "sink") if inf_only.has_node("sink") else []
        raise InfeasibleError(f"sp_ac: forced-save path through {path}") from None
    if cut_value == INF:
        raise InfeasibleError(f"sp_ac plan infeasible under mode {mode.value}")
    saved = [n for n in joint_module.graph.nodes
             if n in fw and n.name + "_in" in reach and n.name + "_out" not in reach]
    saved_sym = [n for n in saved if not isinstance(n.meta.get("val"), torch.Tensor)]
    saved_vals = [n for n in saved if isinstance(n.meta.get("val"), torch.Tensor)]
    recomputed = [n for n in fw if n.op != "placeholder" and n.name + "_out" not in reach]
    guards = [n.name for n in joint_module.graph.nodes if n in fw and guarded(n, mode, fw)]
    stats = {"cut_bytes": int(cut_value), "saved": [n.name for n in saved_vals],
             "guarded": guards,
             "_fw_names": {n.name for n in fw if n.op == "call_function"},
             "saved_bytes": _tensor_bytes([n for n in saved_vals if not _aliases_input(n)]),
             "saved_detail": [(n.name, _opname(n), tuple(n.meta["val"].shape))
                              for n in saved_vals],
             "recomputed_candidates": len(recomputed), "mode": mode.value}
    return saved_vals, saved_sym, stats


LAST_PLAN: dict = {}


def _tensor_bytes(nodes) -> int:
    tot = 0
    for n in nodes:
        v = n.meta.get("val") if isinstance(n, fx.Node) else None
        if isinstance(v, torch.Tensor):
            tot += v.numel() * v.element_size()
    return tot


def _save_all_fits(joint_module, fw_mod, num_fwd_outputs) -> tuple[bool, dict]:
    out = next(n for n in fw_mod.graph.nodes if n.op == "output")
    saved = _tensor_bytes(list(out.args[0])[num_fwd_outputs:])
    primals = [n for n in joint_module.graph.nodes
               if n.op == "placeholder" and "primals" in str(n.target)]
    state = STATE_MULTIPLIER * _tensor_bytes(primals)
    total = torch.cuda.get_device_properties(0).total_memory if torch.cuda.is_available() \
        else 0
    budget = MEMORY_FRACTION * total - state
    return saved * TRANSIENT_MARGIN < budget, {"save_all_bytes": saved, "budget_bytes": int(budget)}


def make_partition_fn(mode: AcMode = AcMode.SEQ_AWARE_NON_ATTENTION):
    from torch._functorch.partitioners import (_extract_fwd_bwd_modules, default_partition,
                                               reordering_to_mimic_autograd_engine)

    def partition(joint_module: fx.GraphModule, _joint_inputs, *, num_fwd_outputs, **kwargs):
        eff = mode
        auto_stats = {}
        if mode is AcMode.AUTO:
            fw_mod, bw_mod = default_partition(joint_module, _joint_inputs,
                                               num_fwd_outputs=num_fwd_outputs, **kwargs)
            fits, auto_stats = _save_all_fits(joint_module, fw_mod, num_fwd_outputs)
            if fits:
                LAST_PLAN.clear()
                LAST_PLAN.update(auto_stats, mode="auto", mode_applied="save-all",
                                 bw_recomputes_attention=False,
                                 fw_collectives=sum(is_autosp_collective(n) for n in fw_mod.graph.nodes),
                                 bw_collectives=sum(is_autosp_collective(n) for n in bw_mod.graph.nodes))
                return fw_mod, bw_mod
            eff = AcMode.SEQ_AWARE_NON_ATTENTION
        saved_vals, saved_sym, stats = plan(joint_module, num_fwd_outputs, eff)
        stats.update(auto_stats, mode=mode.value, mode_applied=eff.value)
        fw_mod, bw_mod = _extract_fwd_bwd_modules(joint_module, saved_vals, saved_sym,
                                                  num_fwd_outputs=num_fwd_outputs)
        # recompute each value just before its first backward use (ref schedule.py:45-85)
        bw_mod = reordering_to_mimic_autograd_engine(bw_mod)
        stats["bw_recomputed_ops"] = sorted({_opname(n) for n in bw_mod.graph.nodes
                                             if n.op == "call_function"})
        # forward nodes re-executed in the backward (the recompute schedule, ref
        # ac_pass.py:187-219): the extracted backward keeps the joint graph's node names
        fw_names = stats.pop("_fw_names")
        stats["recomputed_fw_nodes"] = [n.name for n in bw_mod.graph.nodes
                                        if n.op == "call_function" and n.name in fw_names]
        # every forward a2a has exactly one gradient a2a in backward; more means a
        # forward collective was recomputed (the reference's failure mode, SURVEY finding 2)
        n_fw = sum(is_autosp_collective(n) for n in fw_mod.graph.nodes)
        n_bw = sum(is_autosp_collective(n) for n in bw_mod.graph.nodes)
        stats["fw_collectives"], stats["bw_collectives"] = n_fw, n_bw
        stats["bw_recomputes_attention"] = any(is_autosp_attention(n)
                                               for n in bw_mod.graph.nodes)
        LAST_PLAN.clear()
        LAST_PLAN.update(stats)
        return fw_mod, bw_mod

    return partition
