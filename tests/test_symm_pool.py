"""Host-side logic of the symmetric receive-region allocator (dist.SymmetricPool): slots
are recycled when the handed-out storage dies, first-fit, and two ranks issuing the same
program get identical offsets (the invariant the a2a kernels rely on; a violation traps
in autosp_a2a_wait).  Runs on CPU memory (no kernels)."""

import gc

import pytest
import torch

from paper_2604_27089_b200 import dist as sp_dist
from paper_2604_27089_b200.errors import ValidationError


def _pool(nbytes=1 << 20, P=2, rank=0, backing=None):
    backing = backing if backing is not None else torch.zeros(P, nbytes + 4096, dtype=torch.uint8)
    peers = [(backing[j].data_ptr(), backing[j].data_ptr() + 4096) for j in range(P)]
    return sp_dist.SymmetricPool(nbytes, P, rank, torch.device("cpu"), peers=peers), backing


def test_slots_recycle_when_tensor_dies():
    pool, keep = _pool()
    o1, t1 = pool.alloc(3000)
    o2, t2 = pool.alloc(5000)
    assert (o1, o2) == (0, 3072)
    del t1
    gc.collect()
    o3, t3 = pool.alloc(1000)  # first fit reuses the freed slot
    assert o3 == 0
    o4, t4 = pool.alloc(4000)  # does not fit before o2: goes after it
    assert o4 == 3072 + 5120


def test_views_keep_slot_alive():
    pool, keep = _pool()
    off, base = pool.alloc(4096)
    v = base.view(torch.float32)[10:20]
    del base
    gc.collect()
    off2, _ = pool.alloc(4096)
    assert off2 != off  # the view still references the slot's storage
    del v
    gc.collect()
    off3, _ = pool.alloc(4096)
    assert off3 == off


def test_same_program_same_offsets_on_every_rank():
    backing = torch.zeros(2, (1 << 20) + 4096, dtype=torch.uint8)
    pools = [_pool(rank=r, backing=backing)[0] for r in range(2)]

    def program(pool):
        offs, live = [], []
        for i, n in enumerate([4096, 70000, 1200, 33000, 4096, 9000]):
            off, t = pool.alloc(n)
            offs.append(off)
            live.append(t)
            if i % 2:
                live.pop(0)
                gc.collect()
        return offs

    assert program(pools[0]) == program(pools[1])


def test_exhaustion_is_a_validation_error():
    pool, keep = _pool(nbytes=8192)
    _, a = pool.alloc(4096)
    _, b = pool.alloc(4096)
    with pytest.raises(ValidationError):
        pool.alloc(10)


def test_epochs_increase_by_one():
    pool, keep = _pool()
    assert [pool.next_epoch() for _ in range(3)] == [1, 2, 3]
