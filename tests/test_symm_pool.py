"""Host-side logic of the symmetric receive heap (dist.SymmetricPool): slots are recycled
when the handed-out storage dies, first-fit over segments, identical (segment, offset)
pairs for two ranks issuing the same program (the invariant the a2a kernels rely on; a
violation traps in autosp_a2a_wait), and collective growth by whole segments when nothing
fits.  Runs on CPU memory (no kernels; segment mapping is stubbed)."""

import gc

import pytest
import torch

from paper_2604_27089_b200 import dist as sp_dist
from paper_2604_27089_b200.errors import ValidationError


def _pool(nbytes=1 << 20, P=2, rank=0, backing=None):
    backing = backing if backing is not None else torch.zeros(P, nbytes + 4096, dtype=torch.uint8)
    peers = [(backing[j].data_ptr(), backing[j].data_ptr() + 4096) for j in range(P)]
    return sp_dist.SymmetricPool(nbytes, P, rank, torch.device("cpu"), peers=peers), backing


class _GrowPool(sp_dist.SymmetricPool):
    """A pool whose segments are CPU buffers (one per simulated rank) and whose collective
    mapping step is local: exercises the growth bookkeeping without CUDA IPC."""

    def __init__(self, nbytes, grow, P=2, rank=0):
        self.keep = []
        super().__init__(nbytes, P, rank, torch.device("cpu"), grow_bytes=grow)

    def _map_segment(self, nbytes):
        bufs = [torch.zeros(nbytes, dtype=torch.uint8) for _ in range(self.world)]
        self.keep.append(bufs)
        return [b.data_ptr() for b in bufs]


def test_slots_recycle_when_tensor_dies():
    pool, keep = _pool()
    s1 = pool.alloc(3000)
    s2 = pool.alloc(5000)
    assert (s1.offset, s2.offset) == (0, 3072)
    del s1
    gc.collect()
    s3 = pool.alloc(1000)  # first fit reuses the freed slot
    assert s3.offset == 0
    s4 = pool.alloc(4000)  # does not fit before s2: goes after it
    assert s4.offset == 3072 + 5120


def test_views_keep_slot_alive():
    pool, keep = _pool()
    sl = pool.alloc(4096)
    off = sl.offset
    v = sl.view.view(torch.float32)[10:20]
    del sl
    gc.collect()
    assert pool.alloc(4096).offset != off  # the view still references the slot's storage
    del v
    gc.collect()
    assert pool.alloc(4096).offset == off


def test_alloc_many_one_slot_released_with_last_piece():
    pool, keep = _pool()
    slab = pool.alloc_many([3000, 100, 5000])
    offs = [o for o, _ in slab.pieces]
    assert offs == [0, 3072, 4096] and [v.numel() for _, v in slab.pieces] == [3000, 100, 5000]
    a, b, c = (v for _, v in slab.pieces)
    # one storage per piece: custom ops may not return outputs aliasing each other
    assert len({t.untyped_storage()._cdata for t in (a, b, c)}) == 3
    del slab
    gc.collect()
    del a, b
    gc.collect()
    assert pool.alloc(16).offset != 0  # c keeps the whole slab
    del c
    gc.collect()
    assert pool.alloc(16).offset == 0


def test_same_program_same_offsets_on_every_rank():
    backing = torch.zeros(2, (1 << 20) + 4096, dtype=torch.uint8)
    pools = [_pool(rank=r, backing=backing)[0] for r in range(2)]

    def program(pool):
        offs, live = [], []
        for i, n in enumerate([4096, 70000, 1200, 33000, 4096, 9000]):
            sl = pool.alloc(n)
            offs.append(sl.offset)
            live.append(sl.view)
            if i % 2:
                live.pop(0)
                gc.collect()
        return offs

    assert program(pools[0]) == program(pools[1])


def test_loopback_exhaustion_is_a_validation_error():
    pool, keep = _pool(nbytes=8192)
    a = pool.alloc(4096)
    b = pool.alloc(4096)
    with pytest.raises(ValidationError):
        pool.alloc(10)


def test_heap_grows_by_segments_deterministically():
    """Nothing fits -> a new segment of max(need, grow_bytes); later allocations first-fit
    over all segments in order; two ranks running the same program agree on every
    (segment, offset)."""
    def program(pool):
        out, live = [], []
        for i, n in enumerate([6000, 6000, 20000, 3000, 1000, 50000, 2000]):
            sl = pool.alloc(n)
            out.append((sl.segment, sl.offset))
            live.append(sl.view)
            if i == 3:
                live.pop(0)  # frees the first slot of segment 0
                gc.collect()
        return out, pool

    r0, p0 = program(_GrowPool(8192, 16384, rank=0))
    r1, p1 = program(_GrowPool(8192, 16384, rank=1))
    assert r0 == r1
    assert r0[:3] == [(0, 0), (1, 0), (2, 0)]    # 6000 | 6000 (grow 16K) | 20000 (grow 20K)
    assert r0[3] == (1, 6144)                    # fits after the second 6000
    assert r0[4] == (0, 0)                       # segment 0 freed at i == 3
    assert r0[5][0] == 3 and p0.segments[3].capacity == 50176
    assert p0.capacity == 8192 + 16384 + 20480 + 50176


def test_epochs_increase_by_one():
    pool, keep = _pool()
    assert [pool.next_epoch() for _ in range(3)] == [1, 2, 3]
