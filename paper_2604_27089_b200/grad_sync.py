"""SP-group gradient reduction INSIDE the compiled backward (Listing 1's unchanged
``optimizer.step()``).

Under Ulysses SP every rank holds only a partial gradient of the replicated parameters:
its own tokens' contribution (SURVEY §0 finding 6; the reference's tests sum the
per-rank gradients, test_acceptance.py:89-96).  Instead of an explicit reduction after
``loss.backward()``, ``compile()`` rewrites the AOTAutograd BACKWARD graph: parameter
gradients are grouped into buckets in the order the graph produces them, and right
after the node that completes a bucket an async all-reduce of that bucket is issued
(NCCL on its own stream, so it overlaps the rest of the backward: the last layers'
weight gradients travel while the earlier layers' backward still runs).  One wait node
just before the graph's output joins the collectives, so when ``loss.backward()``
returns every ``p.grad`` is the full gradient, averaged over data-parallel replicas.

The all-reduce runs over the default group = SP groups x DP groups (``dist.init``),
with the bucket pre-scaled by 1/DP: sum over the SP group and mean over DP in ONE
collective.  Parameters of the compiled model that are used OUTSIDE the compiled graphs
(e.g. an LM head applied by an eager loss) are reduced by a post-accumulate-grad hook
instead (async, joined at the end of the backward).  Every parameter of a model compiled
this way is marked ``_autosp_grad_sync``, so ``dist.reduce_gradients`` and
``zero.ShardedAdamW`` do not reduce it a second time.  (A parameter used both inside and
outside the compiled graphs -- tied weights split across the boundary -- is not
supported: its eager partial would not be reduced.)

The AOTAutograd backward returns one gradient per forward input, in input order
(checked at rewrite time); the forward inputs that are ``nn.Parameter`` objects are the
ones reduced (a sequence-sharded input's gradient is per-rank and is left alone)."""

from __future__ import annotations

import operator
import os
import weakref

import torch
import torch.distributed as tdist
import torch.fx

from .errors import ValidationError

BUCKET_BYTES = 64 << 20
COVERED = "_autosp_grad_sync"   # set on every parameter of a model compiled with grad sync
IN_GRAPH = "_autosp_in_graph"   # set on parameters reduced inside a compiled backward
_ACCUMULATED = "_autosp_grad_accumulated"  # this backward's contribution reduced apart
_PENDING: list = []             # (work, param, contribution) issued by the eager hooks
LAST: dict = {}                 # stats of the last rewritten backward graph (tests/tools)


def bucket_bytes() -> int:
    env = os.environ.get("AUTOSP_GRAD_BUCKET_BYTES")
    return int(env) if env else BUCKET_BYTES


def enabled(st) -> bool:
    """In-graph reduction applies when this process is part of a multi-rank job (SP > 1
    or DP > 1) and dist.init did not turn it off."""
    return (tdist.is_initialized() and tdist.get_world_size() > 1 and
            getattr(st, "grad_sync", True))


class GradSync:
    """Runtime state of one compiled backward graph's bucketed reduction."""

    def __init__(self, params: list, dp_size: int):
        self.params = [weakref.ref(p) for p in params]
        self.scale = 1.0 / dp_size
        self.works: list = []

    # ---- called from the rewritten backward graph
    def start(self, *grads):
        flat = torch.cat([g.reshape(-1) for g in grads])
        if self.scale != 1.0:
            flat.mul_(self.scale)
        self.works.append(tdist.all_reduce(flat, async_op=True))
        outs, off = [], 0
        for g in grads:
            n = g.numel()
            outs.append(flat[off:off + n].view(g.shape))
            off += n
        return tuple(outs)

    def finish(self):
        works, self.works = self.works, []
        for w in works:
            w.wait()  # NCCL: the current stream waits for the collective (host does not)


def _graph_fns(sync: GradSync):
    """Plain closures as FX call_function targets (codegen keeps them as globals)."""
    def autosp_grad_bucket_start(*grads):
        return sync.start(*grads)

    def autosp_grad_sync_finish(*_deps):
        sync.finish()

    return autosp_grad_bucket_start, autosp_grad_sync_finish


def insert(bw: torch.fx.GraphModule, param_index: list[int], params: list, n_inputs: int,
           dp_size: int, bucket: int | None = None) -> GradSync | None:
    """Rewrite the backward graph `bw` in place (see module doc).  `param_index[i]` is
    the forward-input position of `params[i]`."""
    if not param_index:
        return None
    g = bw.graph
    out = next(n for n in g.nodes if n.op == "output")
    grads = list(out.args[0])
    if len(grads) != n_inputs:
        raise ValidationError(
            f"in-graph gradient reduction: backward returns {len(grads)} gradients for "
            f"{n_inputs} forward inputs; cannot match them to parameters")
    order = {n: i for i, n in enumerate(g.nodes)}
    items = []  # (position in graph, output slot, param)
    for pi, p in zip(param_index, params):
        gn = grads[pi]
        if isinstance(gn, torch.fx.Node):
            val = gn.meta.get("val")
            nbytes = val.numel() * val.element_size() if isinstance(val, torch.Tensor) else 0
            dt = val.dtype if isinstance(val, torch.Tensor) else None
            items.append((order[gn], pi, gn, nbytes, dt))
    if not items:
        return None
    items.sort(key=lambda t: t[0])
    cap = bucket or bucket_bytes()
    buckets, cur, size = [], [], 0
    for it in items:
        if cur and (size + it[3] > cap or it[4] != cur[0][4]):
            buckets.append(cur)
            cur, size = [], 0
        cur.append(it)
        size += it[3]
    if cur:
        buckets.append(cur)
    sync = GradSync([p for p in params], dp_size)
    for p in params:
        setattr(p, IN_GRAPH, True)
    start_fn, finish_fn = _graph_fns(sync)
    new_grads = list(grads)
    starts = []
    for bk in buckets:
        last = max(bk, key=lambda t: t[0])[2]
        if last.op == "placeholder":  # a gradient passed straight through: start after
            last = [n for n in g.nodes if n.op == "placeholder"][-1]  # the inputs
        with g.inserting_after(last):
            st = g.call_function(start_fn, tuple(t[2] for t in bk))
        starts.append(st)
        prev = st
        for j, t in enumerate(bk):
            with g.inserting_after(prev):
                gi = g.call_function(operator.getitem, (st, j))
            new_grads[t[1]] = gi
            prev = gi
    with g.inserting_before(out):
        g.call_function(finish_fn, tuple(starts))
    out.args = (tuple(new_grads),) + tuple(out.args[1:])
    pos = {n: i for i, n in enumerate(g.nodes)}
    LAST.update(buckets=len(buckets), params=len(items), nodes=len(pos),
                start_positions=[pos[x] for x in starts])
    g.lint()
    bw.recompile()
    return sync


def _join_pending():
    """End of a backward that issued eager reductions: wait for them; an accumulated
    contribution (see install) is added to its parameter's .grad here."""
    items, _PENDING[:] = list(_PENDING), []
    for work, p, contrib in items:
        work.wait()
        if p is not None:
            p.grad.add_(contrib)


def _enqueue(work, p=None, contrib=None):
    if not _PENDING:  # first eager reduction of this backward: join them at its end
        torch.autograd.Variable._execution_engine.queue_callback(_join_pending)
    _PENDING.append((work, p, contrib))


def install(model: torch.nn.Module, dp_size: int) -> None:
    """Mark every parameter of `model` as reduced by the compiled backward, and hook the
    ones that end up used outside it (see module doc).  Idempotent per parameter.

    Eager parameters: the usual case (no .grad yet) reduces the accumulated .grad in
    place after accumulation (post-accumulate hook, async, joined at the end of the
    backward).  Gradient accumulation (.grad already holds earlier micro-batches' reduced
    gradients) must reduce only THIS backward's contribution: the tensor hook takes it,
    starts its reduction on a copy and hands autograd zeros instead; the reduced copy is
    added to .grad when the backward ends."""
    scale = 1.0 / dp_size

    def make_hooks(p):
        def contribution(g):  # before accumulation
            if getattr(p, IN_GRAPH, False) or p.grad is None:
                return None
            red = g * scale if scale != 1.0 else g.clone()
            _enqueue(tdist.all_reduce(red, async_op=True), p, red)
            setattr(p, _ACCUMULATED, True)
            return torch.zeros_like(g)

        def accumulated(p):  # after accumulation
            if getattr(p, IN_GRAPH, False) or p.grad is None:
                return
            if getattr(p, _ACCUMULATED, False):  # reduced separately (contribution)
                setattr(p, _ACCUMULATED, False)
                return
            g = p.grad
            if scale != 1.0:
                g.mul_(scale)
            _enqueue(tdist.all_reduce(g, async_op=True))

        return contribution, accumulated

    for p in model.parameters():
        if p.requires_grad and not getattr(p, COVERED, False):
            setattr(p, COVERED, True)
            contribution, accumulated = make_hooks(p)
            p.register_hook(contribution)
            p.register_post_accumulate_grad_hook(accumulated)


def consume(params) -> list:
    """The parameters (with gradients) of `params` whose gradients are NOT reduced by a
    compiled backward -- what an explicit reduction still has to sum."""
    return [p for p in params if p.grad is not None and not getattr(p, COVERED, False)]
