"""Optimizer step inside the compiled backward (opt_in_bw.py), CPU: the rewrite must place
each parameter's update after the backward's LAST read of that parameter (the input
gradient dX = dY W reads W after dW exists) -- checked against the same SGD update done
after a normal backward, bit for bit, on a model whose weights are read several times
and through views (W.t(), a tied use)."""

import torch

from paper_2604_27089_b200 import compiler


class _SGD:
    """Minimal optimizer with the step_params protocol (optim.AdamW's, CUDA-only)."""

    def __init__(self, params, lr):
        self.param_groups = [{"params": list(params)}]
        self.lr = lr
        self.updated = []

    @torch.no_grad()
    def step_params(self, pairs):
        for p, g in pairs:
            p.sub_(self.lr * g)
            self.updated.append(p)


class _MMWeightGradFirst(torch.autograd.Function):
    """x @ w.t() whose backward computes dW BEFORE it reads w for dX -- the order in
    which an in-graph update placed right after dW would corrupt dX."""

    @staticmethod
    def forward(ctx, x, w):
        ctx.save_for_backward(x, w)
        return x @ w.t()

    @staticmethod
    def backward(ctx, g):
        x, w = ctx.saved_tensors
        dw = g.t() @ x
        dx = g @ w
        return dx, dw


class _Net(torch.nn.Module):
    def __init__(self):
        super().__init__()
        g = torch.Generator().manual_seed(0)
        self.w1 = torch.nn.Parameter(torch.randn(16, 8, generator=g, dtype=torch.float64))
        self.w2 = torch.nn.Parameter(torch.randn(16, 16, generator=g, dtype=torch.float64))
        self.w3 = torch.nn.Parameter(torch.randn(4, 16, generator=g, dtype=torch.float64))

    def forward(self, x):
        h = torch.tanh(x @ self.w1.t())
        h = torch.tanh(_MMWeightGradFirst.apply(h, self.w2))  # dW2 before the dX read of w2
        return (h @ self.w3.t()).pow(2).sum()


def test_in_graph_updates_equal_post_backward_updates():
    torch._dynamo.reset()
    xs = [torch.randn(5, 8, generator=torch.Generator().manual_seed(i), dtype=torch.float64)
          for i in range(3)]
    ref = _Net()
    for x in xs:
        ref(x).backward()
        with torch.no_grad():
            for p in ref.parameters():
                p.sub_(0.01 * p.grad)
                p.grad = None
    net = _Net()
    opt = _SGD(net.parameters(), 0.01)
    cm = torch.compile(net, backend=compiler.backend([], optimizer=opt), dynamic=False)
    for x in xs:
        cm(x).backward()
        assert all(p.grad is None for p in net.parameters())  # no gradient survives
    assert len(opt.updated) == 3 * 3
    for a, b in zip(net.parameters(), ref.parameters()):
        assert torch.equal(a.detach(), b.detach())
    torch._dynamo.reset()
