"""``dist.init(SP_GROUP_SIZE)`` — the Ulysses process-group plumbing (paper Listing 1;
reference equivalent ``DeviceGroup(P)``, ``executor.py:233-275``).

One process per GPU.  The world is split into data-parallel replicas of
``sp_group_size`` consecutive ranks.  Inside an SP group every rank owns one
*symmetric* allocation (identical size on all ranks) holding

    [ flag block (256 B) | receive region ]

mapped once into every peer through CUDA IPC, so the all-to-all kernels write straight
into peers' HBM over NVLink 5 / NVSwitch (no NCCL on the reshard path).  NCCL (or gloo
on CPU test runs) carries only the host-side rendezvous and the per-step gradient
reduction.

Receive-region allocation is deterministic on every rank: a first-fit allocator whose
slots are released when the storage of the tensor handed out is no longer referenced
(C++ refcount, identical on all ranks running the same program).  The kernels verify
at run time that sender and receiver agree on every offset (a mismatch traps)."""

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
POOL_FRACTION = 0.12  # of device memory reserved per rank for a2a receive slots


def default_pool_bytes(device) -> int:
    """The a2a outputs that sp_ac keeps (q/k/v head shards + o seq shard per layer) live in
    the pool until their backward, so size it with the device (override:
    AUTOSP_POOL_BYTES or dist.init(pool_bytes=...))."""
    env = os.environ.get("AUTOSP_POOL_BYTES")
    if env:
        return int(env)
    total = torch.cuda.get_device_properties(device).total_memory
    return int(total * POOL_FRACTION) // (1 << 20) * (1 << 20)


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
    base: torch.Tensor  # uint8 view owned by the pool; busy while its storage is shared


class SymmetricPool:
    """Receive region + flag block of one rank, with the peers' mappings."""

    ALIGN = 1024

    def __init__(self, nbytes: int, world: int, rank: int, device, group=None,
                 peers: list[tuple[int, int]] | None = None, reuse: bool = True):
        lib = _lib.load()
        self.world, self.rank, self.device = world, rank, device
        # reuse=False: bump allocation, no slot reuse -- for virtual ranks sharing ONE
        # process (threads share the autograd engine, so slot lifetimes, and with them
        # first-fit offsets, can differ between ranks; separate processes are symmetric)
        self.reuse = reuse
        self.capacity = nbytes
        self._owned: list[int] = []
        self._opened: list[int] = []
        if peers is None:
            ptr = C.c_void_p()
            handle = (C.c_char * _lib.IPC_HANDLE_BYTES)()
            _lib.check(lib.autosp_symm_alloc(FLAG_BYTES + nbytes, C.byref(ptr), handle),
                       "symm_alloc")
            self._owned.append(ptr.value)
            handles = [None] * world
            if world > 1:
                tdist.all_gather_object(handles, bytes(handle), group=group)
            bases = []
            for j in range(world):
                if j == rank:
                    bases.append(ptr.value)
                else:
                    pp = C.c_void_p()
                    _lib.check(lib.autosp_symm_open(handles[j], C.byref(pp)), "symm_open")
                    self._opened.append(pp.value)
                    bases.append(pp.value)
            self.flag_ptrs = bases
            self.region_ptrs = [b + FLAG_BYTES for b in bases]
        else:  # explicit (flag_ptr, region_ptr) per rank: single-process loopback
            self.flag_ptrs = [f for f, _ in peers]
            self.region_ptrs = [r for _, r in peers]
        self.slots: list[_Slot] = []
        self.epoch = 0
        self.high_water = 0

    # ------------------------------------------------------------------ allocation
    @staticmethod
    def _busy(slot: _Slot) -> bool:
        return torch._C._storage_Use_Count(slot.base.untyped_storage()._cdata) > 2

    def alloc(self, nbytes: int) -> tuple[int, torch.Tensor]:
        """First-fit slot of the receive region; returns (offset, uint8 view)."""
        if not self.reuse:
            need = (nbytes + self.ALIGN - 1) // self.ALIGN * self.ALIGN
            off = self.high_water
            if off + need > self.capacity:
                raise ValidationError("loopback receive region exhausted (bump allocation)")
            self.high_water = off + need
            base = _raw_tensor(self.region_ptrs[self.rank] + off, nbytes, self.device)
            return off, base.view(-1)
        self.slots = [s for s in self.slots if self._busy(s)]
        self.slots.sort(key=lambda s: s.offset)
        need = (nbytes + self.ALIGN - 1) // self.ALIGN * self.ALIGN
        off = 0
        for s in self.slots:
            if s.offset - off >= need:
                break
            off = max(off, s.offset + (s.nbytes + self.ALIGN - 1) // self.ALIGN * self.ALIGN)
        if off + need > self.capacity:
            raise ValidationError(
                f"symmetric receive region exhausted ({off + need} > {self.capacity} bytes); "
                "raise AUTOSP_POOL_BYTES / dist.init(pool_bytes=...)")
        # a separate storage per slot so its C++ refcount tracks exactly this slot
        base = _raw_tensor(self.region_ptrs[self.rank] + off, nbytes, self.device)
        self.slots.append(_Slot(off, nbytes, base))
        self.high_water = max(self.high_water, off + need)
        # hand out a VIEW: the caller's reference then holds the slot's storage (the
        # pool's own `base` alone does not count as busy)
        return off, base.view(-1)

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


_STATE: SPState | None = None
_REGISTRY: dict[str, SPState] = {}


def init(sp_group_size: int, pool_bytes: int | None = None, backend: str | None = None) -> SPState:
    """Create the SP groups (consecutive ranks), map the symmetric receive regions."""
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
    st = SPState(world=sp_group_size, rank=rank % sp_group_size, device=device)
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
        st.pool = SymmetricPool(pool_bytes or default_pool_bytes(device), sp_group_size, st.rank,
                                device, group=st.group)
    _STATE = st
    _REGISTRY[st.name] = st
    return st


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
    is one bucket, not a flat copy of every gradient (16 GB for an 8B model)."""
    st = st or state()
    if not tdist.is_initialized():
        return
    grads = [p.grad for p in params if p.grad is not None]
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
