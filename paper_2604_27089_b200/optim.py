"""AdamW over bf16 parameters with bf16 moments, one multi-tensor sm_100a kernel per 64
tensors (`autosp_adamw_bf16`, csrc/fused.cu).  Drop-in for
``torch.optim.AdamW(params, lr, betas, eps, weight_decay, fused=True)`` on bf16 CUDA
parameters (same update order, fp32 math, bf16 state); the training step the bench
times ends with it.  No CPU path: CUDA bf16 parameters only."""

from __future__ import annotations

import ctypes as C

import torch

from . import _lib
from .errors import ValidationError

UPDATED = "_autosp_updated"  # set by step_params (update done inside the backward)


class _Tensor(C.Structure):
    _fields_ = [("p", C.c_void_p), ("g", C.c_void_p), ("m", C.c_void_p), ("v", C.c_void_p),
                ("n", C.c_int64)]


class AdamW(torch.optim.Optimizer):
    def __init__(self, params, lr: float = 1e-3, betas=(0.9, 0.999), eps: float = 1e-8,
                 weight_decay: float = 1e-2):
        super().__init__(params, dict(lr=lr, betas=betas, eps=eps, weight_decay=weight_decay))
        for group in self.param_groups:
            for p in group["params"]:
                if p.dtype != torch.bfloat16 or not p.is_cuda or not p.is_contiguous():
                    raise ValueError("optim.AdamW: contiguous bf16 CUDA parameters only")

    @torch.no_grad()
    def step(self, closure=None):
        loss = closure() if closure is not None else None
        for group in self.param_groups:
            # parameters the compiled backward already updated in this iteration
            # (autosp.compile(model, optimizer=...)) are skipped once
            live = []
            for p in group["params"]:
                if getattr(p, UPDATED, False):
                    setattr(p, UPDATED, False)
                    if p.grad is not None:  # a gradient from outside the compiled graph
                        raise ValidationError(
                            "optim.AdamW: a parameter updated inside the compiled backward "
                            "also has a .grad from code outside it (a weight shared between "
                            "the compiled model and eager code) -- not supported with "
                            "compile(optimizer=...)")
                elif p.grad is not None:
                    live.append(p)
            self._apply(group, [(p, p.grad) for p in live])
        return loss

    @torch.no_grad()
    def step_params(self, pairs) -> None:
        """AdamW on the given (parameter, gradient) pairs right now -- called from inside
        a compiled backward graph (optimizer in the backward: the gradient is freed as
        soon as its parameter is updated); the next ``step()`` skips these parameters.
        ``step()`` must run once per iteration (Listing 1's loop): a second in-backward
        update of a parameter before it means two compiled graphs both own the parameter
        (a weight shared across a graph break), each with a partial gradient -- refused."""
        for group in self.param_groups:
            mine = [(p, g) for p, g in pairs if any(p is q for q in group["params"])]
            for p, _ in mine:
                if getattr(p, UPDATED, False):
                    raise ValidationError(
                        "optim.AdamW: parameter updated twice inside the backward before "
                        "step(): either step() was not called after the last iteration, or "
                        "the parameter is used by two compiled graphs (shared across a graph "
                        "break) -- not supported with compile(optimizer=...)")
            if mine:
                self._apply(group, mine)
                for p, _ in mine:
                    setattr(p, UPDATED, True)

    def _apply(self, group, pairs) -> None:
        lib = _lib.load()
        stream = torch.cuda.current_stream().cuda_stream
        if pairs:
            live = [p for p, _ in pairs]
            grads = {id(p): g for p, g in pairs}
            # the bias corrections depend on each parameter's own step count: one launch
            # per distinct step value (normally exactly one)
            by_step: dict[int, list] = {}
            for p in live:
                st = self.state[p]
                if not st:
                    st["step"] = 0
                    st["exp_avg"] = torch.zeros_like(p)
                    st["exp_avg_sq"] = torch.zeros_like(p)
                st["step"] += 1
                g = grads[id(p)]
                g = g if g.is_contiguous() else g.contiguous()
                if g.dtype != torch.bfloat16:
                    raise ValueError("optim.AdamW: bf16 gradients only")
                st["_g"] = g  # keep a made-contiguous gradient alive until the launch
                by_step.setdefault(st["step"], []).append(p)
            b1, b2 = group["betas"]
            for step, ps in by_step.items():
                arr = (_Tensor * len(ps))()
                for i, p in enumerate(ps):
                    st = self.state[p]
                    arr[i] = _Tensor(p.data_ptr(), st["_g"].data_ptr(), st["exp_avg"].data_ptr(),
                                     st["exp_avg_sq"].data_ptr(), p.numel())
                rc = lib.autosp_adamw_bf16(arr, len(ps), group["lr"], b1, b2, group["eps"],
                                           group["weight_decay"], step, stream)
                _lib.check(rc, "adamw_bf16")
                from .kernels import LOG
                LOG.end("adamw", None, (len(ps) + 63) // 64)
            for p in live:
                self.state[p].pop("_g", None)
