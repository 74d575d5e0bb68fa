"""ZeRO-1 over the SP group: the SP-group gradient reduction fused with optimizer-state
sharding (the paper trains with ZeRO-1; the reference
models optimizer state as a static memory term only, cost_model.py:121-123).

The parameters of a model are viewed as one flat vector (in ``params`` order, padded to
a multiple of the SP size P) cut into chunks of at most ``bucket_bytes``.  Rank r owns
slice r of every chunk.  ``step()``:

  1. per chunk: the per-rank partial gradients (Ulysses SP produces partials, finding 6)
     are packed and reduce-scattered over the SP group -> this rank's summed shard
     (averaged over the DP group when there is one);
  2. AdamW on the owned shards only (optim.AdamW for bf16 on CUDA, torch otherwise) -- optimizer
     state is 1/P of the model per rank;
  3. the updated shards are all-gathered back into the full parameters.

Same bytes on the wire as an all-reduce; 2·(P-1)/P of the optimizer-state memory freed
(for Llama-3-8B with bf16 AdamW state at P = 8: 32 GB -> 4 GB per GPU).  AdamW is
elementwise, so the result equals unsharded AdamW on the summed gradients."""

from __future__ import annotations

import torch
import torch.distributed as tdist

from . import grad_sync
from .dist import SPState, state


class ShardedAdamW:
    def __init__(self, params, st: SPState | None = None, bucket_bytes: int = 256 << 20,
                 **adamw_kwargs):
        self.params = [p for p in params if p.requires_grad]
        self.st = st or state()
        P = self.st.world if (self.st.group is not None and self.st.world > 1) else 1
        self.P, self.rank = P, (self.st.rank if P > 1 else 0)
        self.group = self.st.group if P > 1 else None
        dp = self.st.dp_group
        self.dp = dp if (dp is not None and tdist.is_initialized() and
                         tdist.get_world_size(dp) > 1) else None
        p0 = self.params[0]
        self.dtype, self.device = p0.dtype, p0.device
        if any(p.dtype != self.dtype for p in self.params):
            raise ValueError("ShardedAdamW: all parameters must share one dtype")
        self.sizes = [p.numel() for p in self.params]
        total = sum(self.sizes)
        elems = max(P, (bucket_bytes // p0.element_size()) // P * P)
        padded = (total + P - 1) // P * P
        self.chunks = [(a, min(a + elems, padded)) for a in range(0, padded, elems)]
        self.total = total
        # owned shard of every chunk (a copy of the parameter values), optimised by AdamW
        self.shards = []
        for a, b in self.chunks:
            n = (b - a) // P
            lo = a + self.rank * n
            sh = torch.nn.Parameter(self._gather_params(lo, lo + n))
            self.shards.append(sh)
        kw = dict(adamw_kwargs)
        if self.device.type == "cuda" and self.dtype == torch.bfloat16:
            from .optim import AdamW  # the multi-tensor bf16 kernel
            self.inner = AdamW(self.shards, **kw)
        else:
            if self.device.type == "cuda":
                kw.setdefault("fused", True)
            self.inner = torch.optim.AdamW(self.shards, **kw)

    # -------------------------------------------------------------- flat-vector helpers
    def _pieces(self, lo: int, hi: int):
        """(param index, start, stop) element ranges of the flat interval [lo, hi)."""
        off = 0
        for i, n in enumerate(self.sizes):
            a, b = max(lo, off), min(hi, off + n)
            if a < b:
                yield i, a - off, b - off
            off += n
            if off >= hi:
                break

    def _gather_params(self, lo: int, hi: int) -> torch.Tensor:
        out = torch.zeros(hi - lo, dtype=self.dtype, device=self.device)
        pos = 0
        for i, a, b in self._pieces(lo, hi):
            out[pos:pos + b - a].copy_(self.params[i].detach().reshape(-1)[a:b])
            pos += b - a
        return out

    def _flat_grads(self, lo: int, hi: int) -> torch.Tensor:
        out = torch.zeros(hi - lo, dtype=self.dtype, device=self.device)
        pos = 0
        for i, a, b in self._pieces(lo, hi):
            g = self.params[i].grad
            if g is not None:
                out[pos:pos + b - a].copy_(g.reshape(-1)[a:b])
            pos += b - a
        return out

    def _scatter_back(self, flat: torch.Tensor, lo: int, hi: int) -> None:
        pos = 0
        with torch.no_grad():
            for i, a, b in self._pieces(lo, hi):
                self.params[i].view(-1)[a:b].copy_(flat[pos:pos + b - a])
                pos += b - a

    # -------------------------------------------------------------- collectives
    def _reduce_scatter(self, flat: torch.Tensor, out: torch.Tensor) -> None:
        # (the same collectives on NCCL and on gloo, so the CPU tests run this code)
        if self.P == 1:
            out.copy_(flat)
        else:
            tdist.reduce_scatter_tensor(out, flat, group=self.group)
        if self.dp is not None:
            tdist.all_reduce(out, group=self.dp)
            out /= tdist.get_world_size(self.dp)

    def _all_gather(self, shard: torch.Tensor, flat: torch.Tensor) -> None:
        if self.P == 1:
            flat.copy_(shard)
        else:
            tdist.all_gather_into_tensor(flat, shard, group=self.group)

    # -------------------------------------------------------------- optimizer API
    @torch.no_grad()
    def step(self) -> None:
        # gradients the compiled backward already all-reduced (grad_sync.py) are full
        # sums: take this rank's slice instead of reduce-scattering them again
        todo = grad_sync.consume(self.params)
        reduced = not todo or len(todo) < sum(p.grad is not None for p in self.params)
        if reduced and todo:  # a mix: bring the rest to full sums too
            from .dist import reduce_gradients
            reduce_gradients(todo, self.st)
        for (a, b), sh in zip(self.chunks, self.shards):
            n = (b - a) // self.P
            g = torch.empty(n, dtype=self.dtype, device=self.device)
            if reduced:
                g.copy_(self._flat_grads(a + self.rank * n, a + (self.rank + 1) * n))
            else:
                self._reduce_scatter(self._flat_grads(a, b), g)  # (zero padding past the end)
            sh.grad = g
        self.inner.step()
        for (a, b), sh in zip(self.chunks, self.shards):
            sh.grad = None
            flat = torch.empty(b - a, dtype=self.dtype, device=self.device)
            self._all_gather(sh.detach(), flat)
            self._scatter_back(flat, a, b)

    def zero_grad(self, set_to_none: bool = True) -> None:
        for p in self.params:
            if set_to_none:
                p.grad = None
            elif p.grad is not None:
                p.grad.zero_()

    def state_bytes(self) -> int:
        """Optimizer state held by THIS rank (the owned shards + their AdamW moments)."""
        tot = 0
        for sh in self.shards:
            tot += sh.numel() * sh.element_size()
            for v in self.inner.state.get(sh, {}).values():
                if isinstance(v, torch.Tensor):
                    tot += v.numel() * v.element_size()
        return tot
