"""Optimizer step inside the compiled backward on the Llama block (optim.AdamW, the bf16
multi-tensor kernel), one GPU.

* Bit-exact given the same gradients: every gradient the compiled backward hands to the
  optimizer (and the eager LM head's, updated by step()) is recorded, and replaying them
  through the normal loop (p.grad = g; optimizer.step()) from the same initial weights
  gives BIT-IDENTICAL parameters after two steps.  (Comparing two independent training
  runs bit for bit is not possible: the attention backward accumulates dQ over key tiles
  with fp32 atomics, whose order -- and so the last bit -- varies run to run, as in
  FlashAttention; tools/bwd_determinism.py measures it.)
* Against an independent normal run the parameters agree up to that noise.
* Every compiled parameter is updated inside the graph (only the eager LM head by
  step()), and when the backward returns the compiled parameters' gradients are already
  gone (the memory the normal loop holds until step())."""

import pytest
import torch

pytestmark = pytest.mark.gpu

_LR = 1e-3


def _run(in_backward: bool, mode: str):
    import paper_2604_27089_b200 as autosp
    from paper_2604_27089_b200 import opt_in_bw
    from paper_2604_27089_b200.optim import AdamW
    from paper_2604_27089_b200.workloads import LlamaConfig, LlamaDecoder, lm_loss
    torch._dynamo.reset()
    cfg = LlamaConfig("oib", 512, 2, 8, 4, 1024, 2048)
    autosp.reg_passes(["auto_sp", "sp_ac"], ac_mode=mode)
    autosp.dist.init(1)
    torch.manual_seed(0)
    model = LlamaDecoder(cfg, dtype=torch.bfloat16, device="cuda")
    init = [p.detach().clone() for p in model.parameters()]
    index = {id(p): i for i, p in enumerate(model.parameters())}
    opt = AdamW(model.parameters(), lr=_LR)
    recorded = []  # per step: {param index: gradient}
    inner = opt.step_params

    def recording_step_params(pairs):
        for p, g in pairs:
            recorded[-1][index[id(p)]] = g.detach().clone()
        inner(pairs)

    opt.step_params = recording_step_params
    cm = autosp.compile(model, optimizer=opt if in_backward else None)
    g = torch.Generator().manual_seed(3)
    peaks, after_bwd = [], []
    for _ in range(2):
        recorded.append({})
        ids = torch.randint(0, cfg.vocab, (1, 4097), generator=g).cuda()
        torch.cuda.synchronize()
        torch.cuda.reset_peak_memory_stats()
        loss = lm_loss(cm(ids[:, :-1]), model.lm_head, ids[:, 1:])
        loss.backward()
        torch.cuda.synchronize()
        peaks.append(torch.cuda.max_memory_allocated())
        after_bwd.append(torch.cuda.memory_allocated())
        n_grads = sum(p.grad is not None for p in model.parameters())
        for p in model.parameters():  # what step() will apply
            if p.grad is not None:
                recorded[-1][index[id(p)]] = p.grad.detach().clone()
        opt.step()
        opt.zero_grad(set_to_none=True)
    torch.cuda.synchronize()
    params = [p.detach().clone() for p in model.parameters()]
    torch._dynamo.reset()
    grad_bytes = sum(p.numel() * p.element_size() for p in model.parameters()
                     if p is not model.lm_head)
    return (params, init, recorded), (peaks, after_bwd, grad_bytes), n_grads, \
        dict(opt_in_bw.LAST)


def _replay(init, recorded):
    """The normal loop (gradients in .grad, then optimizer.step()) fed the recorded
    gradients, from the same initial weights."""
    from paper_2604_27089_b200.optim import AdamW
    params = [torch.nn.Parameter(t.clone()) for t in init]
    opt = AdamW(params, lr=_LR)
    for grads in recorded:
        assert len(grads) == len(params)
        for i, p in enumerate(params):
            p.grad = grads[i]
        opt.step()
        opt.zero_grad(set_to_none=True)
    torch.cuda.synchronize()
    return [p.detach() for p in params]


@pytest.mark.parametrize("mode", ["seq-aware", "auto"])
def test_optimizer_in_backward_bit_exact_and_frees_gradients(mode):
    (ref, _, _), ref_peaks, ref_grads, _ = _run(False, mode)
    (got, init, recorded), peaks, n_grads, info = _run(True, mode)
    for a, b in zip(got, _replay(init, recorded)):  # same gradients -> same bits
        assert torch.equal(a, b)
    for a, b, a0 in zip(got, ref, init):  # independent normal run: equal up to the dQ
        upd = (a.float() - a0.float()).norm()  # atomics (last-bit flips of the updates)
        assert (a.float() - b.float()).norm() <= 0.1 * upd, ((a != b).float().mean(), upd)
    assert info["updated_in_graph"] == 2 * 6 + 2  # 6 weights per block + embedding + norm
    assert n_grads == 1 and ref_grads == 2 * 6 + 3  # only the eager LM head keeps a .grad
    (pk_ref, ab_ref, gbytes), (pk, ab, _) = ref_peaks, peaks
    print("after backward (normal, in-backward):", ab_ref[-1], ab[-1], "peak:", pk_ref[-1], pk[-1])
    if mode == "auto":  # save-all: nothing recomputed, the gradients are all that is freed
        assert ab[-1] <= ab_ref[-1] - 0.9 * gbytes, (ab, ab_ref, gbytes)


class _Tiny(torch.nn.Module):
    def __init__(self):
        super().__init__()
        self.w = torch.nn.Parameter(torch.randn(32, 32, device="cuda").bfloat16())

    def forward(self, x):
        return (x @ self.w.t()).float().pow(2).sum()


def _tiny_compiled():
    from paper_2604_27089_b200 import compiler
    from paper_2604_27089_b200.optim import AdamW
    torch._dynamo.reset()
    net = _Tiny()
    opt = AdamW(net.parameters(), lr=1e-3)
    cm = torch.compile(net, backend=compiler.backend([], optimizer=opt), dynamic=False)
    return net, opt, cm, torch.randn(8, 32, device="cuda").bfloat16()


def test_weight_shared_with_eager_code_is_refused():
    """A parameter updated inside the backward that ALSO got an eager gradient (a weight
    shared between the compiled model and eager code) would lose that gradient: step()
    refuses."""
    from paper_2604_27089_b200.errors import ValidationError
    net, opt, cm, x = _tiny_compiled()
    (cm(x) + net.w.float().sum()).backward()
    with pytest.raises(ValidationError, match="outside"):
        opt.step()
    torch._dynamo.reset()


def test_second_update_without_step_is_refused():
    """step() runs once per iteration (Listing 1); a second in-backward update before it
    (or a parameter owned by two compiled graphs) is refused, not applied twice."""
    from paper_2604_27089_b200.errors import ValidationError
    net, opt, cm, x = _tiny_compiled()
    cm(x).backward()
    opt.step()
    cm(x).backward()  # fine: step() ran in between
    with pytest.raises(Exception, match="updated twice"):
        cm(x).backward()
    torch._dynamo.reset()
