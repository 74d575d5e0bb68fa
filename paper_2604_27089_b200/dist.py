"""``dist.init(SP_GROUP_SIZE)`` — the Ulysses process-group plumbing (paper Listing 1;
reference equivalent ``DeviceGroup(P)``, ``executor.py:233-275``).

One process per GPU.  The world is split into data-parallel replicas of
``sp_group_size`` consecutive ranks.  Inside an SP group every rank owns a *symmetric*
heap: segments of identical size on all ranks, the first one holding

    [ flag block (256 B used of 4 KB) | receive region ]

each mapped into every peer through CUDA IPC, so the all-to-all kernels write straight
into peers' HBM over NVLink 5 / NVSwitch (no NCCL on the reshard path).  NCCL (or gloo
on CPU test runs) carries only the host-side rendezvous (the IPC handles of a new
segment) and the per-step gradient reduction.

Receive-heap allocation is deterministic on every rank: first-fit over the segments,
slots released when the storage of the tensor handed out is no longer referenced (C++
refcount, identical on all ranks running the same program), and the heap grows
collectively when nothing fits.  Every call's destination descriptors are folded into a
check word the receiver compares with each sender's (a mismatch traps)."""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import torch
import torch.distributed as tdist
import torch.utils.dlpack

from . import _lib
from .errors import ValidationError

FLAG_BYTES = 4096  # flag block (256 B used) padded to keep the receive region aligned
POOL_INITIAL_BYTES = 2 << 30  # first segment of the symmetric receive heap
POOL_GROW_BYTES = 2 << 30     # minimum size of each further segment (the heap grows on demand)
SPIN_TIMEOUT_S = 300.0  # default bound of a flag spin (AUTOSP_SPIN_TIMEOUT_S overrides)


def default_pool_bytes(device) -> int:
    """Initial size of the symmetric heap's first segment (it grows on demand; override:
    AUTOSP_POOL_BYTES or dist.init(pool_bytes=...), e.g. planner.pool_bytes(cfg, S, P) to
    get the whole steady-state heap in one segment)."""
    env = os.environ.get("AUTOSP_POOL_BYTES")
    if env:
        return int(env)
    return POOL_INITIAL_BYTES


def default_grow_bytes() -> int:
    env = os.environ.get("AUTOSP_POOL_GROW_BYTES")
    return int(env) if env else POOL_GROW_BYTES


_PyCapsule_New = C.pythonapi.PyCapsule_New
_PyCapsule_New.restype = C.py_object
_PyCapsule_New.argtypes = [C.c_void_p, C.c_char_p, C.c_void_p]


def _raw_tensor(ptr: int, nbytes: int, device) -> torch.Tensor:
    """Zero-copy uint8 tensor over raw device memory we own (its own StorageImpl, no
    allocator involvement and -- unlike __cuda_array_interface__ -- no stream sync).  The
    DLPack struct is allocated and freed in C (autosp_dlpack_wrap), so dropping the view
    never calls back into Python (a Python deleter segfaulted at interpreter shutdown)."""
    dev = torch.device(device)
    cuda = dev.type == "cuda"
    mt = _lib.load().autosp_dlpack_wrap(ptr, nbytes, 2 if cuda else 1,
                                        (dev.index or 0) if cuda else 0)
    if not mt:
        _lib.check(2, "dlpack_wrap")
    return torch.utils.dlpack.from_dlpack(_PyCapsule_New(mt, b"dltensor", None))


@dataclass
class _Slot:
    offset: int
    nbytes: int
    # uint8 views owned by the pool, one storage per piece handed out; the slot is busy
    # while ANY of those storages is still shared with a caller
    bases: list[torch.Tensor]


@dataclass
class Slab:
    """One allocation of the symmetric heap: `view` (uint8, this rank's memory) sits at
    byte `offset` of segment `segment`, whose receive region rank j maps at regions[j]
    -- the same offset on every rank, so a sender addresses rank j's copy as
    regions[j] + offset."""
    segment: int
    offset: int
    view: torch.Tensor
    regions: list[int]

    pieces: list[tuple[int, torch.Tensor]] = field(default_factory=list)


def _align(n: int) -> int:
    return (n + SymmetricPool.ALIGN - 1) // SymmetricPool.ALIGN * SymmetricPool.ALIGN


class _Segment:
    def __init__(self, capacity: int, regions: list[int]):
        self.capacity = capacity
        self.regions = regions
        self.slots: list[_Slot] = []
        self.high_water = 0


class SymmetricPool:
    """Symmetric receive heap of one rank: a list of SEGMENTS, each one cudaMalloc per rank
    mapped into every peer through CUDA IPC; segment 0 also holds the flag block.

    Allocation is first-fit over the segments in order, slots are released when the
    storage of the tensor handed out is no longer referenced (C++ refcount), so ranks
    running the same program get identical (segment, offset) pairs.  When no segment has
    room, the heap GROWS collectively: every rank reaches the same failing allocation at
    the same point of the program, allocates a new segment of max(need, grow_bytes), and
    the SP group exchanges the IPC handles (all_gather_object) -- so the receive heap is
    sized by what sp_ac actually keeps (the q/k/v head shards and token-major O of every
    layer until its backward), not by a fixed fraction of the device."""

    ALIGN = 1024

    def __init__(self, nbytes: int, world: int, rank: int, device, group=None,
                 peers: list[tuple[int, int]] | None = None, reuse: bool = True,
                 grow_bytes: int | None = None):
        self.world, self.rank, self.device, self.group = world, rank, device, group
        # reuse=False: bump allocation, no slot reuse -- for virtual ranks sharing ONE
        # process (threads share the autograd engine, so slot lifetimes, and with them
        # first-fit offsets, can differ between ranks; separate processes are symmetric)
        self.reuse = reuse
        self.grow_bytes = grow_bytes if grow_bytes is not None else default_grow_bytes()
        self._owned: list[int] = []
        self._opened: list[int] = []
        self.segments: list[_Segment] = []
        if peers is None:
            bases = self._map_segment(FLAG_BYTES + nbytes)
            if bases is None:
                raise torch.OutOfMemoryError(f"symmetric heap: cannot allocate {nbytes} bytes")
            self.flag_ptrs = bases
            self.segments.append(_Segment(nbytes, [b + FLAG_BYTES for b in bases]))
            self.growable = True
        else:  # explicit (flag_ptr, region_ptr) per rank: single-process loopback
            self.flag_ptrs = [f for f, _ in peers]
            self.segments.append(_Segment(nbytes, [r for _, r in peers]))
            self.growable = False
        self.epoch = 0

    # ------------------------------------------------------------------ segments
    def _map_segment(self, nbytes: int) -> list[int] | None:
        """Collective: allocate `nbytes` on every rank and map all peers' allocations.
        Returns the per-rank base pointers, or None on every rank if ANY rank failed."""
        lib = _lib.load()
        ptr = C.c_void_p()
        handle = (C.c_char * _lib.IPC_HANDLE_BYTES)()
        rc = lib.autosp_symm_alloc(nbytes, C.byref(ptr), handle)
        if rc != 0 and self.device.type == "cuda":
            torch.cuda.empty_cache()  # cached-but-free blocks of the caching allocator
            rc = lib.autosp_symm_alloc(nbytes, C.byref(ptr), handle)
        mine = (rc == 0, bytes(handle))
        allh = [None] * self.world
        if self.world > 1 and tdist.is_initialized():
            tdist.all_gather_object(allh, mine, group=self.group)
        else:
            allh = [mine] * self.world
        if not all(ok for ok, _ in allh):
            if rc == 0:
                lib.autosp_symm_free(ptr.value)
            return None
        self._owned.append(ptr.value)
        bases = []
        for j in range(self.world):
            if j == self.rank:
                bases.append(ptr.value)
            else:
                pp = C.c_void_p()
                _lib.check(lib.autosp_symm_open(allh[j][1], C.byref(pp)), "symm_open")
                self._opened.append(pp.value)
                bases.append(pp.value)
        return bases

    @property
    def region_ptrs(self) -> list[int]:
        """Segment 0's receive regions (rank j's, as mapped here)."""
        return self.segments[0].regions

    @property
    def capacity(self) -> int:
        return sum(sg.capacity for sg in self.segments)

    @property
    def high_water(self) -> int:
        return sum(sg.high_water for sg in self.segments)

    # ------------------------------------------------------------------ allocation
    @staticmethod
    def _busy(slot: _Slot) -> bool:
        return any(torch._C._storage_Use_Count(b.untyped_storage()._cdata) > 2
                   for b in slot.bases)

    def _fit(self, sg: _Segment, need: int) -> int | None:
        if not self.reuse:
            return sg.high_water if sg.high_water + need <= sg.capacity else None
        sg.slots = [x for x in sg.slots if self._busy(x)]
        sg.slots.sort(key=lambda x: x.offset)
        off = 0
        for x in sg.slots:
            if x.offset - off >= need:
                break
            off = max(off, x.offset + _align(x.nbytes))
        return off if off + need <= sg.capacity else None

    def alloc(self, nbytes: int, sizes: list[int] | None = None) -> Slab:
        """First-fit slab of `nbytes` (growing the heap collectively if nothing fits)."""
        need = _align(max(nbytes, 1))
        for i, sg in enumerate(self.segments):
            off = self._fit(sg, need)
            if off is not None:
                return self._take(i, off, nbytes, need, sizes)
        if not (self.growable and self.reuse):
            raise ValidationError(
                f"symmetric receive region exhausted ({need} bytes requested, "
                f"{self.capacity} total); loopback pools do not grow")
        cap = max(need, self.grow_bytes)
        bases = self._map_segment(cap)
        if bases is None:
            raise torch.OutOfMemoryError(
                f"symmetric heap: growing by {cap} bytes failed on some rank of the SP group "
                f"(heap {self.capacity} bytes in {len(self.segments)} segments)")
        self.segments.append(_Segment(cap, bases))
        return self._take(len(self.segments) - 1, 0, nbytes, need, sizes)

    def _take(self, i: int, off: int, nbytes: int, need: int,
              sizes: list[int] | None = None) -> Slab:
        sg = self.segments[i]
        # a separate storage per piece so the C++ refcounts track exactly this slot and
        # the pieces of one call do not alias each other (custom ops may not return
        # aliasing outputs)
        many = sizes is not None
        sizes = [nbytes] if sizes is None else sizes
        bases, pieces, cur = [], [], 0
        for n in sizes:
            bases.append(_raw_tensor(sg.regions[self.rank] + off + cur, max(n, 1), self.device))
            # hand out VIEWS: the caller's reference then holds the piece's storage (the
            # pool's own base alone does not count as busy)
            pieces.append((off + cur, bases[-1].view(-1)[:n]))
            cur += _align(n)
        if self.reuse:
            sg.slots.append(_Slot(off, need, bases))
        sg.high_water = max(sg.high_water, off + need)
        slab = Slab(i, off, pieces[0][1], sg.regions)
        if many:
            slab.pieces = pieces
        return slab

    def alloc_many(self, sizes: list[int]) -> Slab:
        """One slab holding consecutive ALIGN-aligned pieces of the given sizes (the
        destinations of one call, all in one segment so one peer-base array addresses
        them; slab.pieces = [(offset, uint8 view)], each piece its own storage).  The
        slot is released when the last piece dies."""
        return self.alloc(sum(_align(n) for n in sizes), sizes=sizes)

    def next_epoch(self) -> int:
        self.epoch += 1
        return self.epoch

    def close(self):
        lib = _lib.load()
        for p in self._opened:
            lib.autosp_symm_close(p)
        for p in self._owned:
            lib.autosp_symm_free(p)
        self._opened, self._owned = [], []


@dataclass
class SPState:
    world: int = 1               # SP group size P
    rank: int = 0                # rank inside the SP group
    group: object = None         # torch ProcessGroup of the SP group (None when P == 1)
    dp_group: object = None      # data-parallel group of this rank's SP position
    device: torch.device = field(default_factory=lambda: torch.device("cpu"))
    pool: SymmetricPool | None = None
    name: str = "sp"
    grad_sync: bool = True       # compile() all-reduces parameter gradients in-graph


_STATE: SPState | None = None
_REGISTRY: dict[str, SPState] = {}


def init(sp_group_size: int, pool_bytes: int | None = None, backend: str | None = None,
         grad_sync: bool = True) -> SPState:
    """Create the SP groups (consecutive ranks), map the symmetric receive regions.

    grad_sync (default): models compiled afterwards reduce their parameter gradients
    inside the backward graph (sum over the SP group, mean over DP; grad_sync.py), so
    the training loop stays ``loss.backward(); optimizer.step()``.  With False the loop
    must call ``reduce_gradients`` (or use ``zero.ShardedAdamW``)."""
    global _STATE
    if sp_group_size < 1:
        raise ValidationError("sp_group_size must be positive")
    if not tdist.is_initialized():
        if int(os.environ.get("WORLD_SIZE", "1")) > 1 or sp_group_size > 1:
            be = backend or ("nccl" if torch.cuda.is_available() else "gloo")
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29511")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
            tdist.init_process_group(be)
    world = tdist.get_world_size() if tdist.is_initialized() else 1
    rank = tdist.get_rank() if tdist.is_initialized() else 0
    if world % sp_group_size:
        raise ValidationError(f"world size {world} not divisible by SP group size {sp_group_size}")
    if torch.cuda.is_available():
        # (modulo: several ranks may share a device in single-GPU multi-process tests)
        local = int(os.environ.get("LOCAL_RANK", rank)) % max(torch.cuda.device_count(), 1)
        torch.cuda.set_device(local)
        device = torch.device("cuda", local)
    else:
        device = torch.device("cpu")
    st = SPState(world=sp_group_size, rank=rank % sp_group_size, device=device,
                 grad_sync=grad_sync)
    if tdist.is_initialized() and world > 1:
        for g0 in range(0, world, sp_group_size):
            ranks = list(range(g0, g0 + sp_group_size))
            pg = tdist.new_group(ranks)
            if rank in ranks:
                st.group = pg
        for r0 in range(sp_group_size):
            ranks = list(range(r0, world, sp_group_size))
            pg = tdist.new_group(ranks)
            if rank in ranks:
                st.dp_group = pg
    if sp_group_size > 1 and device.type == "cuda":
        # bound of the reshard protocol's flag spins (a peer that never arrives traps the
        # kernel instead of hanging the GPU); compile skew is absorbed by the host barrier
        # before each compiled graph's first run (compiler.py), not by this timeout
        _lib.check(_lib.load().autosp_set_spin_timeout(
            float(os.environ.get("AUTOSP_SPIN_TIMEOUT_S", SPIN_TIMEOUT_S))), "set_spin_timeout")
        st.pool = SymmetricPool(pool_bytes or default_pool_bytes(device), sp_group_size, st.rank,
                                device, group=st.group)
    _STATE = st
    _REGISTRY[st.name] = st
    return st


def barrier(st: SPState | None = None) -> None:
    """Host barrier over the SP group (no-op without a process group)."""
    st = st or state()
    if st.group is not None and st.world > 1 and tdist.is_initialized():
        tdist.barrier(group=st.group)


def state() -> SPState:
    if _STATE is None:
        return SPState()
    return _STATE


def lookup(name: str) -> SPState:
    try:
        return _REGISTRY[name]
    except KeyError:
        raise ValidationError(f"SP group {name!r} is not initialised (call dist.init)") from None


def register_state(st: SPState) -> None:
    """Used by single-process loopback harnesses (tests / bench) to install a state."""
    global _STATE
    _STATE = st
    _REGISTRY[st.name] = st


REDUCE_BUCKET_BYTES = 128 << 20


def reduce_gradients(params, st: SPState | None = None,
                     bucket_bytes: int = REDUCE_BUCKET_BYTES) -> None:
    """Sum the per-rank partial parameter gradients over the SP group (SURVEY §0 finding 6:
    the reference's tests sum them, test_acceptance.py:89-96) and average over DP.
    Gradients are packed into buckets of at most ``bucket_bytes`` (one collective per
    bucket; a gradient larger than a bucket is reduced in place), so the transient memory
    is one bucket, not a flat copy of every gradient (16 GB for an 8B model).
    Gradients already reduced inside a compiled backward (grad_sync.py) are skipped."""
    from . import grad_sync
    st = st or state()
    if not tdist.is_initialized():
        return
    grads = [p.grad for p in grad_sync.consume(params)]
    if not grads:
        return
    sp = st.group if (st.group is not None and st.world > 1) else None
    dp = st.dp_group if (st.dp_group is not None and tdist.get_world_size(st.dp_group) > 1) \
        else None
    if sp is None and dp is None:
        return

    def reduce(t):
        if sp is not None:
            tdist.all_reduce(t, group=sp)
        if dp is not None:
            tdist.all_reduce(t, group=dp)
            t /= tdist.get_world_size(dp)

    def flush(bucket):
        if not bucket:
            return
        if len(bucket) == 1:
            reduce(bucket[0])
            return
        flat = torch.cat([g.reshape(-1) for g in bucket])
        reduce(flat)
        off = 0
        for g in bucket:
            n = g.numel()
            g.copy_(flat[off:off + n].view_as(g))
            off += n

    bucket, size = [], 0
    for g in grads:
        nb = g.numel() * g.element_size()
        if bucket and (size + nb > bucket_bytes or g.dtype != bucket[0].dtype):
            flush(bucket)
            bucket, size = [], 0
        bucket.append(g)
        size += nb
    flush(bucket)
