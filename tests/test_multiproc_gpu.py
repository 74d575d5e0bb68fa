"""Two PROCESSES, one GPU: the real multi-process AutoSP path — `dist.init(2)` exchanging
CUDA IPC handles of the symmetric receive regions (all_gather_object), the push kernels
writing into the peer process's mapped memory with the epoch-flag protocol, AOTAutograd
graphs from auto_sp + sp_ac, and the SP-group gradient reduction — on a Llama-shaped
model, compared with the same model run unsharded (P = 1) in a third process.

Only the transport differs from a multi-GPU run (both ranks' peer pointers resolve to
the same device instead of NVLink peers).  gloo carries the host-side rendezvous and the
gradient all-reduce because NCCL refuses two ranks on one device.
Tolerances (north star): loss rel 1e-3, gradients max|g-g_ref|/max|g_ref| 2e-2."""

import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

CFG = dict(d_model=256, layers=2, hq=4, hkv=2, d_ffn=512, vocab=512)
CFG4 = dict(d_model=512, layers=2, hq=8, hkv=4, d_ffn=1024, vocab=512)  # heads divisible by 4
SEQ = 1024


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mode, q, cfgd=None):
    import torch.distributed as tdist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK="0", AUTOSP_POOL_BYTES=str(64 << 20))
    try:
        if world > 1:
            tdist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2604_27089_b200 as autosp
        from paper_2604_27089_b200 import sp_ac
        from paper_2604_27089_b200.workloads import LlamaConfig, LlamaDecoder, lm_loss
        c = cfgd or CFG
        cfg = LlamaConfig("mp", c["d_model"], c["layers"], c["hq"], c["hkv"], c["d_ffn"],
                          c["vocab"])
        autosp.reg_passes(["auto_sp", "sp_ac"], ac_mode=mode)
        st = autosp.dist.init(world)
        torch.manual_seed(0)
        model = LlamaDecoder(cfg, dtype=torch.bfloat16, device="cuda")
        cm = autosp.compile(model)
        g = torch.Generator().manual_seed(7)
        ids = torch.randint(0, cfg.vocab, (1, SEQ + 1), generator=g)
        sl = SEQ // world
        x = ids[:, rank * sl:(rank + 1) * sl].cuda()
        y = ids[:, rank * sl + 1:(rank + 1) * sl + 1].cuda()
        loss = lm_loss(cm(x), model.lm_head, y)
        loss.backward()
        params = list(model.parameters())
        if world > 1:
            # Listing 1's loop: no explicit reduction -- the compiled backward all-reduced
            # the SP-partial gradients (grad_sync.py; lm_head, used outside the compiled
            # graph by the eager loss, through its post-accumulate hook)
            from paper_2604_27089_b200 import grad_sync
            assert not grad_sync.consume(params)
            lt = torch.tensor([float(loss)])
            tdist.all_reduce(lt)
            total = float(lt)
        else:
            total = float(loss)
        torch.cuda.synchronize()
        grads = {n: p.grad.float().cpu().numpy() for n, p in model.named_parameters()}
        from paper_2604_27089_b200 import compiler
        info = compiler.LAST_INFO.get("auto_sp")
        q.put((rank, total, grads, sp_ac.LAST_PLAN.get("fw_collectives"),
               sp_ac.LAST_PLAN.get("bw_collectives"), info.fused_qkv_proj if info else 0))
        if world > 1:
            tdist.barrier()
    except Exception:
        import traceback
        q.put((rank, "ERROR", traceback.format_exc(), None, None, None))
    finally:
        if world > 1 and tdist.is_initialized():
            tdist.destroy_process_group()


def _run(world, mode, cfgd=None):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, q, cfgd))
             for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        item = q.get(timeout=600)
        res[item[0]] = item
    for p in procs:
        p.join(timeout=120)
    for item in res.values():
        assert item[1] != "ERROR", item[2]
    return [res[r] for r in range(world)]


@pytest.mark.parametrize("mode", ["seq-aware", "auto"])
def test_two_processes_ipc_match_unsharded(mode):
    ref = _run(1, mode)[0]
    out = _run(2, mode)
    _, ref_loss, ref_grads, _, _, _ = ref
    for rank, loss, grads, n_fw, n_bw, n_proj in out:
        # the QKV projection GEMM itself pushes RoPE'd head-major rows (K0) in every layer
        assert n_proj == CFG["layers"], n_proj
        assert abs(loss - ref_loss) / abs(ref_loss) < 1e-3, (loss, ref_loss)
        # forward: ONE collective op per layer (QKV GEMM pushing RoPE'd q/k/v + attention
        # whose epilogue pushes O); backward: TWO (dO reshard fused with delta =
        # rowsum(dO * O); the attention backward pushing dq/dk/dv from its epilogues)
        assert n_fw == CFG["layers"] and n_bw == 2 * CFG["layers"]
        for n, gr in ref_grads.items():
            err = float(abs(grads[n] - gr).max() / max(abs(gr).max(), 1e-30))
            assert err < 2e-2, (rank, n, err)


def test_four_processes_ipc_match_unsharded():
    """P = 4 ranks as four processes on one GPU (each rank pushes into three peers'
    mapped regions), seq-aware sp_ac, K0 / K3 / K4 pushes and the dO + delta reshard."""
    ref = _run(1, "seq-aware", CFG4)[0]
    out = _run(4, "seq-aware", CFG4)
    _, ref_loss, ref_grads, _, _, _ = ref
    for rank, loss, grads, n_fw, n_bw, n_proj in out:
        assert n_proj == CFG4["layers"], n_proj
        assert abs(loss - ref_loss) / abs(ref_loss) < 1e-3, (loss, ref_loss)
        assert n_fw == CFG4["layers"] and n_bw == 2 * CFG4["layers"]
        for n, gr in ref_grads.items():
            err = float(abs(grads[n] - gr).max() / max(abs(gr).max(), 1e-30))
            assert err < 2e-2, (rank, n, err)
