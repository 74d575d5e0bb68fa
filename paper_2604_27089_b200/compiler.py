"""``reg_passes([...])`` and ``compile(model)`` — the paper's user API (Listing 1,
PAPER.md:62-72) over torch.compile used as a graph-capture front end only:

  Dynamo FX graph --auto_sp--> Torch IR with autosp ops --AOTAutograd--> joint graph
  --sp_ac partitioner--> forward / backward graphs executed eagerly (boxed), whose hot
  ops are the sm_100a kernels in libautosp.so; everything else is plain ATen/cuBLAS.

No Inductor, no Triton: the compiled graphs run their ATen ops and our custom ops
directly.  Reference equivalents: SPConfig + transform_sp (sp_pass.py:57-68,133-220),
AcMode + plan_checkpoints (ac_pass.py:26-29,181-184)."""

from __future__ import annotations

import functools
import os

import torch
import torch.distributed as tdist

from . import dist as sp_dist
from . import grad_sync, opt_in_bw
from .auto_sp import auto_sp
from .errors import ValidationError
from .sp_ac import AcMode, is_autosp_collective, make_partition_fn

KNOWN_PASSES = ("auto_sp", "sp_ac")
_PASSES: list[str] = []
_AC_MODE = AcMode.AUTO
LAST_INFO: dict = {}
_COMPILER_OVERRIDE = None  # debug tools (tools/mem_trace.py) swap in a tracing executor


def reg_passes(passes: list[str], ac_mode: str | AcMode = AcMode.AUTO) -> None:
    global _AC_MODE
    unknown = [p for p in passes if p not in KNOWN_PASSES]
    if unknown:
        raise ValidationError(f"unknown passes {unknown}; known: {list(KNOWN_PASSES)}")
    if "sp_ac" in passes and "auto_sp" not in passes:
        raise ValidationError("sp_ac requires auto_sp")
    _PASSES[:] = list(passes)
    _AC_MODE = AcMode(ac_mode)


def registered_passes() -> list[str]:
    return list(_PASSES)


def backend(passes: list[str] | None = None, ac_mode: AcMode | None = None, optimizer=None):
    """A torch.compile backend applying the registered passes."""
    from functorch.compile import make_boxed_func
    from torch._dynamo.backends.common import aot_autograd
    from torch._functorch.partitioners import default_partition

    passes = list(_PASSES if passes is None else passes)
    mode = _AC_MODE if ac_mode is None else AcMode(ac_mode)

    def _compiler(gm, example_inputs, sync=None, opt=None):
        if _COMPILER_OVERRIDE is not None:
            return _COMPILER_OVERRIDE(gm, example_inputs)
        if sync is not None:  # backward graph: bucketed SP/DP gradient all-reduce
            grad_sync.insert(gm, *sync)
        if opt is not None:  # backward graph: parameters updated as their gradients appear
            opt_in_bw.insert(gm, *opt)
        fn = make_boxed_func(gm.forward)
        st = sp_dist.state()
        if st.world > 1 and st.group is not None and \
                any(is_autosp_collective(n) for n in gm.graph.nodes):
            # every rank compiles the same graphs in the same order but not at the same
            # speed: a host barrier before a graph's FIRST run keeps one rank's first
            # reshard from spinning on a peer that is still compiling
            first = [True]

            def fn_sync(args):
                if first[0]:
                    first[0] = False
                    sp_dist.barrier(st)
                return fn(args)

            fn_sync._boxed_call = True
            return fn_sync
        return fn

    def _backend(gm: torch.fx.GraphModule, example_inputs):
        st = sp_dist.state()
        if "auto_sp" in passes:
            gm, info = auto_sp(gm, example_inputs, st)
            LAST_INFO["auto_sp"] = info
        base_part = make_partition_fn(mode) if "sp_ac" in passes else default_partition
        aliases: dict = {}

        def part(joint_module, joint_inputs, **kw):
            if optimizer is not None:  # which joint nodes are views of which parameter
                aliases.update(opt_in_bw.alias_names(joint_module))
            return base_part(joint_module, joint_inputs, **kw)

        bw = _compiler
        if optimizer is not None:
            pidx = [i for i, x in enumerate(example_inputs) if isinstance(x, torch.nn.Parameter)]
            bw = functools.partial(_compiler, opt=(pidx, [example_inputs[i] for i in pidx],
                                                   len(example_inputs), aliases, optimizer))
        if grad_sync.enabled(st):
            # the forward inputs that are parameters: their (partial) gradients are
            # all-reduced inside the backward graph, overlapped with it (grad_sync.py)
            pidx = [i for i, x in enumerate(example_inputs) if isinstance(x, torch.nn.Parameter)]
            dp = tdist.get_world_size() // max(st.world, 1)
            sync = (pidx, [example_inputs[i] for i in pidx], len(example_inputs), dp)
            bw = functools.partial(_compiler, sync=sync)
            if optimizer is not None:
                raise ValidationError("optimizer in the backward needs a single rank (the "
                                      "SP-partial gradients are reduced at the graph's end)")
        return aot_autograd(fw_compiler=_compiler, bw_compiler=bw,
                            partition_fn=part)(gm, example_inputs)

    return _backend


def _frames():
    from torch._dynamo.utils import counters
    f = counters["frames"]
    return f.get("total", 0), f.get("ok", 0)


def compile(model: torch.nn.Module, passes: list[str] | None = None,
            ac_mode: AcMode | None = None, optimizer=None) -> torch.nn.Module:
    """``model.compile()`` with the AutoSP backend (static shapes).

    Graph breaks are allowed (``fullgraph=False``): auto_sp rewrites every Dynamo
    subgraph, including attention-free ones.  But a frame Dynamo gives up on (e.g. a
    graph break inside a loop: "skipping the frame and falling back to eager") would run
    its attention eagerly over the LOCAL shard only -- silently wrong at P > 1.  So at
    P > 1 a call that left any frame uncompiled raises ValidationError (set
    AUTOSP_ALLOW_EAGER_FRAMES=1 if the skipped frames are known to hold no attention).

    optimizer (opt-in, single rank): an ``optim.AdamW`` that updates each parameter INSIDE
    the compiled backward as soon as its gradient exists (opt_in_bw.py): the gradients are
    never all alive at once; ``optimizer.step()`` then handles only the parameters used
    outside the compiled graphs."""
    passes_eff = list(_PASSES if passes is None else passes)
    st = sp_dist.state()
    if grad_sync.enabled(st):  # SP-partial gradients summed by the backward itself
        grad_sync.install(model, tdist.get_world_size() // max(st.world, 1))
    if optimizer is not None and not hasattr(optimizer, "step_params"):
        raise ValidationError("compile(optimizer=...) needs an optimizer with step_params "
                              "(optim.AdamW)")
    cm = torch.compile(model, backend=backend(passes, ac_mode, optimizer), dynamic=False,
                       fullgraph=False)
    if "auto_sp" not in passes_eff:
        return cm
    snap = {}

    def pre(_mod, _args):
        snap["f"] = _frames()

    def post(_mod, _args, _out):
        t0, ok0 = snap.pop("f", (0, 0))
        t1, ok1 = _frames()
        if (t1 - t0) > (ok1 - ok0) and sp_dist.state().world > 1 and \
                os.environ.get("AUTOSP_ALLOW_EAGER_FRAMES") != "1":
            raise ValidationError(
                f"{(t1 - t0) - (ok1 - ok0)} frame(s) of the model fell back to eager execution "
                "(a graph break inside a loop?): attention there would not be sequence-"
                "parallel.  Move the graph break out of the loop (or set "
                "AUTOSP_ALLOW_EAGER_FRAMES=1 if those frames hold no attention).")

    cm.register_forward_pre_hook(pre)
    cm.register_forward_hook(post)
    return cm
