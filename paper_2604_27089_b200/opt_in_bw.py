"""Optimizer step inside the compiled backward (opt-in: ``compile(model, optimizer=opt)``).

A training step normally holds every weight gradient until ``optimizer.step()``: for the
Llama-3-8B shape that is 16 GB of bf16 gradients on top of the activations saved for the
backward, at the point of the step where memory peaks.  Here the AOTAutograd backward
graph is rewritten so that each parameter is updated (``optim.AdamW.step_params``: the same
multi-tensor AdamW kernel, same math) as soon as its gradient exists AND the backward has
finished reading the parameter, and the graph returns no gradient for it -- the gradient
dies right there.  ``optimizer.step()`` afterwards only updates parameters the compiled
graph does not own (e.g. an LM head applied by an eager loss).  The result is the same
parameters, bit for bit (``tests/test_opt_in_bw_gpu.py``); peak memory drops by up to the
gradient bytes, which extends the single-GPU trainable context (BASELINE.json configs[3]).

"Finished reading" is found by data flow: the backward graph's inputs are named after the
joint graph's nodes, the parameter is joint input ``primals_{i+1}``, and every forward
view of it (``t``, ``view``, ``permute`` ...) that was saved for the backward is followed
through its users in the backward graph; the update is placed after the last of them.

Single SP rank only (SP-partial gradients would first need the all-reduce, which
grad_sync joins at the end of the graph)."""

from __future__ import annotations

import weakref

import torch
import torch.fx as fx

from .errors import ValidationError

_aten = torch.ops.aten
VIEW_OPS = {_aten.t.default, _aten.view.default, _aten._unsafe_view.default,
            _aten.permute.default, _aten.transpose.int, _aten.expand.default,
            _aten.alias.default, _aten.detach.default, _aten.slice.Tensor,
            _aten.select.int, _aten.unsqueeze.default, _aten.squeeze.dim,
            _aten.reshape.default, _aten.as_strided.default}
LAST: dict = {}


def alias_names(joint: fx.GraphModule) -> dict[int, set[str]]:
    """forward input index -> names of the joint-graph nodes that are views of it."""
    root: dict[fx.Node, int] = {}
    out: dict[int, set[str]] = {}
    for n in joint.graph.nodes:
        if n.op == "placeholder" and str(n.target).startswith("primals_"):
            i = int(str(n.target).split("_")[1]) - 1
            root[n] = i
            out[i] = {n.name}
        elif n.op == "call_function" and n.target in VIEW_OPS and n.args and \
                isinstance(n.args[0], fx.Node) and n.args[0] in root:
            root[n] = root[n.args[0]]
            out[root[n]].add(n.name)
    return out


def _readers(start: fx.Node) -> list[fx.Node]:
    """Every node reading `start` or a view of it (views followed transitively)."""
    seen, todo, readers = {start}, [start], []
    while todo:
        x = todo.pop()
        for u in x.users:
            if u in seen:
                continue
            seen.add(u)
            readers.append(u)
            if u.op == "call_function" and u.target in VIEW_OPS:
                todo.append(u)
    return readers


def insert(bw: fx.GraphModule, param_index: list[int], params: list, n_inputs: int,
           aliases: dict[int, set[str]], optimizer) -> int:
    """Rewrite the backward graph in place; returns the number of parameters updated
    inside it."""
    g = bw.graph
    out = next(n for n in g.nodes if n.op == "output")
    grads = list(out.args[0])
    if len(grads) != n_inputs:
        raise ValidationError(f"optimizer in backward: {len(grads)} gradients for {n_inputs} "
                              "forward inputs")
    order = {n: i for i, n in enumerate(g.nodes)}
    placeholders = {n.name: n for n in g.nodes if n.op == "placeholder"}
    owned = {id(q) for grp in optimizer.param_groups for q in grp["params"]}
    done = 0
    for pi, p in zip(param_index, params):
        gn = grads[pi]
        if not isinstance(gn, fx.Node) or id(p) not in owned:
            continue
        last = gn
        for name in aliases.get(pi, ()):
            ph = placeholders.get(name)
            if ph is None:
                continue
            for r in _readers(ph):
                if r.op != "output" and order[r] > order[last]:
                    last = r
        pref = weakref.ref(p)

        def autosp_update_param(grad, pref=pref):
            param = pref()
            if param is not None:
                optimizer.step_params([(param, grad)])

        if last.op == "placeholder":
            last = [n for n in g.nodes if n.op == "placeholder"][-1]
        with g.inserting_after(last):
            g.call_function(autosp_update_param, (gn,))
        grads[pi] = None
        done += 1
    out.args = (tuple(grads),) + tuple(out.args[1:])
    g.lint()
    bw.recompile()
    LAST.update(updated_in_graph=done)
    return done
