"""Multi-GPU paths (one process per GPU, torch.distributed for the plumbing).

* Batches of independent strings (configs 1-4) shard by string with no
  data-path collective: ``shard_round_robin`` / ``shard_blocks``.
* One huge string (config 5) splits at multiples of 8^c instances.  The
  reference's stack construction groups blocks front-aligned
  (halftimehash/tree.py:63-100), so each slice reduces to independent level-c
  subtree roots; finalize terms (tree.py:103-134) and the Toeplitz tail
  (hasher.py:186-206) are sums, so each slice also yields a partial digest.
  The only exchange is gathering the roots (<= a few hundred KB) and the
  partials to rank 0, which finishes the tree with ``hth_hash_merge``.
  Three forms:

  - ``FlagExchange`` (default on distinct GPUs): entirely in-stream.  The
    slice kernels store roots and partials straight into rank 0's memory
    over NVLink (CUDA-IPC peer pointers) and their last warp raises a
    per-rank arrival flag (system-scope release); rank 0's merge kernel
    waits on the flags in-stream, merges, and hands the double-buffered slot
    back through a "consumed" flag the producers wait on before reusing it.
    No host synchronisation or collective on the data path.
  - ``hash_string_p2p``: the same peer stores, then a host synchronize and a
    barrier before rank 0 merges (for ranks sharing one GPU, where kernels
    must never wait on one another).
  - ``hash_string_distributed``: an NCCL ``all_gather`` of roots/partials.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .hasher import SeedBuffer, _check_capacity
from .params import HashParams


@dataclass(frozen=True)
class SlicePlan:
    params: HashParams
    n_bytes: int
    level: int  # frontier level c
    bounds: tuple  # n_slices + 1 instance bounds (multiples of 8^c but the last)
    counts: tuple  # frontier roots emitted by each slice

    @property
    def n_slices(self) -> int:
        return len(self.counts)

    @property
    def n_frontier(self) -> int:
        return sum(self.counts)

    def byte_range(self, i: int):
        """Bytes [b0, b1) of the string that slice i reads."""
        ib = self.params.instance_words * 8
        b0 = self.bounds[i] * ib
        b1 = self.n_bytes if i == self.n_slices - 1 else self.bounds[i + 1] * ib
        return b0, b1


def slice_plan(params: HashParams, n_bytes: int, n_slices: int) -> SlicePlan:
    b = (ctypes.c_uint64 * (n_slices + 1))()
    lvl = ctypes.c_int()
    cnt = (ctypes.c_uint64 * n_slices)()
    _lib.check(_lib.lib().hth_slice_plan(params.output_bytes, n_bytes, n_slices, b, ctypes.byref(lvl), cnt))
    return SlicePlan(params, n_bytes, lvl.value, tuple(int(x) for x in b), tuple(int(x) for x in cnt))


def shard_round_robin(n_strings: int, rank: int, world: int) -> np.ndarray:
    """Config 4: string s goes to rank s % world."""
    return np.arange(rank, n_strings, world)


def shard_blocks(n_strings: int, rank: int, world: int) -> range:
    """Config 3: contiguous index ranges."""
    lo = n_strings * rank // world
    hi = n_strings * (rank + 1) // world
    return range(lo, hi)


_WS = {}


def _ws(dev, nbytes):
    import torch

    t = _WS.get(dev.index)
    if t is None or t.numel() < nbytes:
        t = torch.zeros(max(nbytes, 256), dtype=torch.uint8, device=dev)
        _WS[dev.index] = t
    return t


def hash_slice(data, plan: SlicePlan, i: int, seed: SeedBuffer):
    """Hash slice i on data's GPU.  ``data``: CUDA uint8 tensor holding bytes
    plan.byte_range(i).  Returns (frontier (count, 8k) int64, partial (k,) int64)."""
    import torch

    p = plan.params
    _check_capacity(seed, p, plan.n_bytes)
    dev = data.device
    k = p.output_words
    fr = torch.empty((max(plan.counts[i], 1), 8 * k), dtype=torch.int64, device=dev)
    part = torch.empty(k, dtype=torch.int64, device=dev)
    wsz = ctypes.c_uint64()
    _lib.check(_lib.lib().hth_workspace_size_slice(p.output_bytes, plan.n_bytes, ctypes.byref(wsz)))
    ws = _ws(dev, wsz.value)
    b0, b1 = plan.byte_range(i)
    if data.numel() < b1 - b0:
        raise ValueError("slice tensor shorter than its byte range")
    with torch.cuda.device(dev):
        st = torch.cuda.current_stream(dev).cuda_stream
        _lib.check(_lib.lib().hth_hash_slice(
            p.output_bytes, data.data_ptr(), plan.n_bytes, plan.bounds[i], plan.bounds[i + 1], plan.level, seed.fold,
            seed.device_words(dev).data_ptr(), seed.capacity, fr.data_ptr(), part.data_ptr(), ws.data_ptr(),
            ws.numel(), st))
    return fr[:plan.counts[i]], part


def hash_merge(frontier, partials, plan: SlicePlan, seed: SeedBuffer):
    """Finish the tree from the gathered frontier (n_frontier, 8k) and partials (n, k)."""
    import torch

    p = plan.params
    dev = frontier.device if frontier.numel() else partials.device
    k = p.output_words
    out = torch.empty(k, dtype=torch.int64, device=dev)
    need = 2 * (plan.n_frontier // 8 + 8) * 8 * k * 8
    tmp = torch.empty(need, dtype=torch.uint8, device=dev)
    fr = frontier.contiguous()
    pa = partials.contiguous()
    with torch.cuda.device(dev):
        st = torch.cuda.current_stream(dev).cuda_stream
        _lib.check(_lib.lib().hth_hash_merge(
            p.output_bytes, plan.n_bytes, plan.level, fr.data_ptr() if fr.numel() else None, plan.n_frontier,
            pa.data_ptr(), pa.shape[0], seed.fold, seed.device_words(dev).data_ptr(), seed.capacity,
            out.data_ptr(), tmp.data_ptr(), tmp.numel(), st))
    return out


def hash_string_distributed(local, plan: SlicePlan, seed: SeedBuffer, group=None, slice_fn=None, merge_fn=None):
    """Each rank hashes slice `rank` of one string; rank 0 returns the (k,)
    digest words (numpy uint64), other ranks None.

    The exchange is one all_gather of the padded frontier roots and one of the
    partials (NCCL over NVLink on GPUs; gloo on CPU tensors in the tests).
    ``slice_fn(local, plan, i, seed) -> (frontier, partial)`` and
    ``merge_fn(frontier, partials, plan, seed) -> digest`` default to the CUDA
    engine."""
    import torch
    import torch.distributed as dist

    slice_fn = slice_fn or hash_slice
    merge_fn = merge_fn or hash_merge
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    if world != plan.n_slices:
        raise ValueError("plan must have one slice per rank")
    k = plan.params.output_words
    fr, part = slice_fn(local, plan, rank, seed)
    maxc = max(max(plan.counts), 1)
    pad = torch.zeros((maxc, 8 * k), dtype=torch.int64, device=part.device)
    if fr.shape[0]:
        pad[:fr.shape[0]] = fr
    frs = [torch.empty_like(pad) for _ in range(world)]
    parts = [torch.empty_like(part) for _ in range(world)]
    dist.all_gather(frs, pad, group=group)
    dist.all_gather(parts, part, group=group)
    if rank != 0:
        return None
    frontier = torch.cat([frs[i][:plan.counts[i]] for i in range(world)], dim=0)
    digest = merge_fn(frontier, torch.stack(parts), plan, seed)
    return digest.cpu().numpy().view(np.uint64).copy()


# ------------------------------------------------------------------ peer-memory exchange
_P2P = {}


def _ipc_handle(ptr: int):
    """(64-byte handle of the allocation holding ptr, ptr's offset in it)"""
    h = ctypes.create_string_buffer(64)
    off = ctypes.c_uint64()
    _lib.check(_lib.lib().hth_ipc_get_handle(ptr, h, ctypes.byref(off)))
    return h.raw, int(off.value)


_IPC_OPEN = {}  # allocation handle -> mapped base (a process maps each allocation once)


def _ipc_open(handle) -> int:
    raw, off = handle
    base = _IPC_OPEN.get(raw)
    if base is None:
        buf = ctypes.create_string_buffer(raw, 64)
        out = ctypes.c_void_p()
        _lib.check(_lib.lib().hth_ipc_open_handle(buf, ctypes.byref(out)))
        base = _IPC_OPEN[raw] = int(out.value)
    return base + off


def _p2p_buffers(plan: SlicePlan, dev, group):
    """Rank 0's two gather buffers (double-buffered across calls), mapped into
    every rank: [frontier roots of all slices in slice order | one partial
    digest per slice].  Returns (local tensors or None, base addresses)."""
    import torch
    import torch.distributed as dist

    rank = dist.get_rank(group)
    key = (plan, dev.index, id(group))
    ent = _P2P.get(key)
    if ent is not None:
        return ent
    k = plan.params.output_words
    words = plan.n_frontier * 8 * k + plan.n_slices * k
    buf, handle = None, None
    if rank == 0:
        # both slots in one tensor: one IPC handle (a process maps a handle once)
        buf = torch.zeros(2 * max(words, 1), dtype=torch.int64, device=dev)
        handle = _ipc_handle(buf.data_ptr())
    obj = [handle]
    dist.broadcast_object_list(obj, src=0, group=group)
    b0 = buf.data_ptr() if rank == 0 else _ipc_open(obj[0])
    bases = [b0, b0 + 8 * max(words, 1)]
    bufs = [buf[:max(words, 1)], buf[max(words, 1):]] if rank == 0 else None
    ent = {"bufs": bufs, "bases": bases, "words": words, "step": 0}
    _P2P[key] = ent
    return ent


def hash_string_p2p(local, plan: SlicePlan, seed: SeedBuffer, group=None):
    """Like ``hash_string_distributed`` but without a collective on the data
    path: slice i's kernel (hth_hash_slice) writes its subtree roots and its
    partial digest directly into rank 0's gather buffer through a CUDA-IPC
    peer mapping (NVLink stores), then one barrier; rank 0 merges.  Rank 0
    returns the (k,) digest words (numpy uint64), other ranks None.  The two
    gather buffers alternate, so a rank may start the next string while rank 0
    still merges this one."""
    import torch
    import torch.distributed as dist

    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    if world != plan.n_slices:
        raise ValueError("plan must have one slice per rank")
    p = plan.params
    _check_capacity(seed, p, plan.n_bytes)
    k = p.output_words
    dev = local.device
    ent = _p2p_buffers(plan, dev, group)
    slot = ent["step"] & 1
    ent["step"] += 1
    base = ent["bases"][slot]
    nfw = plan.n_frontier * 8 * k
    fr_ptr = base + sum(plan.counts[:rank]) * 8 * k * 8
    part_ptr = base + (nfw + rank * k) * 8
    wsz = ctypes.c_uint64()
    _lib.check(_lib.lib().hth_workspace_size_slice(p.output_bytes, plan.n_bytes, ctypes.byref(wsz)))
    ws = _ws(dev, wsz.value)
    b0, b1 = plan.byte_range(rank)
    if local.numel() < b1 - b0:
        raise ValueError("slice tensor shorter than its byte range")
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev)
        _lib.check(_lib.lib().hth_hash_slice(
            p.output_bytes, local.data_ptr(), plan.n_bytes, plan.bounds[rank], plan.bounds[rank + 1], plan.level,
            seed.fold, seed.device_words(dev).data_ptr(), seed.capacity, fr_ptr, part_ptr, ws.data_ptr(),
            ws.numel(), stream.cuda_stream))
        stream.synchronize()  # this slice's roots and partial are in rank 0's memory
    dist.barrier(group=group)
    if rank != 0:
        return None
    g = ent["bufs"][slot]
    digest = hash_merge(g[:nfw].view(plan.n_frontier, 8 * k), g[nfw:nfw + world * k].view(world, k), plan, seed)
    return digest.cpu().numpy().view(np.uint64).copy()


# ------------------------------------------------------------ in-stream flag exchange
class _SlotLayout:
    """Word layout of rank 0's exchange buffer (u64 words):
    slot s in {0, 1}: frontier roots [n_frontier, 8k] | partials [n_slices, k];
    then flags [2, n_slices] and consumed [2]."""

    def __init__(self, plan: SlicePlan):
        self.k = plan.params.output_words
        self.n = plan.n_slices
        self.nfw = plan.n_frontier * 8 * self.k
        self.slot_words = self.nfw + self.n * self.k
        self.words = 2 * self.slot_words + 2 * self.n + 2
        self.first = [sum(plan.counts[:r]) for r in range(self.n)]

    def frontier(self, base, slot, r):
        return base + (slot * self.slot_words + self.first[r] * 8 * self.k) * 8

    def partials(self, base, slot, r=0):
        return base + (slot * self.slot_words + self.nfw + r * self.k) * 8

    def flag(self, base, slot, r=0):
        return base + (2 * self.slot_words + slot * self.n + r) * 8

    def consumed(self, base, slot):
        return base + (2 * self.slot_words + 2 * self.n + slot) * 8


def _device_ids(dev, group):
    import torch
    import torch.distributed as dist

    props = torch.cuda.get_device_properties(dev)
    mine = str(getattr(props, "uuid", "")) or f"{props.name}:{dev.index}"
    ids = [None] * dist.get_world_size(group)
    dist.all_gather_object(ids, mine, group=group)
    return ids


class FlagExchange:
    """One split string per ``step`` with the exchange entirely in-stream
    (see the module docstring).  Rank 0's ``step`` returns the (k,) digest
    words as a device tensor (valid once its stream reaches that point);
    ``check()`` synchronizes and raises if any wait timed out.  Requires one
    GPU per rank: a waiting kernel must only wait on another device."""

    def __init__(self, plan: SlicePlan, seed: SeedBuffer, device, group=None, timeout_s: float = 10.0):
        import torch
        import torch.distributed as dist

        self.plan, self.seed, self.group = plan, seed, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        if self.world != plan.n_slices:
            raise ValueError("plan must have one slice per rank")
        self.dev = torch.device(device)
        ids = _device_ids(self.dev, group)
        if len(set(ids)) != len(ids):
            raise RuntimeError("ranks share a GPU: in-stream flag waits would make kernels on one device wait "
                               "on one another; use hash_string_p2p or hash_string_distributed")
        _check_capacity(seed, plan.params, plan.n_bytes)
        self.lay = _SlotLayout(plan)
        self.timeout_ns = int(timeout_s * 1e9)
        self.status_t = torch.zeros(1, dtype=torch.int32, device=self.dev)
        wsz = ctypes.c_uint64()
        _lib.check(_lib.lib().hth_workspace_size_slice(plan.params.output_bytes, plan.n_bytes, ctypes.byref(wsz)))
        self.ws = torch.zeros(max(wsz.value, 256), dtype=torch.uint8, device=self.dev)
        handle = None
        if self.rank == 0:
            self.buf = torch.zeros(self.lay.words, dtype=torch.int64, device=self.dev)
            handle = _ipc_handle(self.buf.data_ptr())
            k = self.lay.k
            self.out = torch.zeros((2, k), dtype=torch.int64, device=self.dev)
            self.mtmp = torch.empty(2 * (plan.n_frontier // 8 + 8) * 8 * k * 8, dtype=torch.uint8, device=self.dev)
        obj = [handle]
        dist.broadcast_object_list(obj, src=0, group=group)
        torch.cuda.synchronize(self.dev)  # rank 0's zeroed buffer exists before any peer store
        dist.barrier(group=group)
        self.base = self.buf.data_ptr() if self.rank == 0 else _ipc_open(obj[0])
        self.epoch = 0

    def step(self, local):
        """Enqueue this rank's slice of one string (and, on rank 0, the merge)."""
        import torch

        plan, lay, L = self.plan, self.lay, _lib.lib()
        p = plan.params
        self.epoch += 1
        e, slot, r = self.epoch, (self.epoch - 1) & 1, self.rank
        b0, b1 = plan.byte_range(r)
        if local.numel() < b1 - b0:
            raise ValueError("slice tensor shorter than its byte range")
        with torch.cuda.device(self.dev):
            st = torch.cuda.current_stream(self.dev).cuda_stream
            if r != 0 and e > 2:  # rank 0 has merged this slot's previous string
                _lib.check(L.hth_wait_flag(lay.consumed(self.base, slot), e - 2, self.timeout_ns,
                                           self.status_t.data_ptr(), st))
            _lib.check(L.hth_hash_slice_ex(
                p.output_bytes, local.data_ptr(), plan.n_bytes, plan.bounds[r], plan.bounds[r + 1], plan.level,
                self.seed.fold, self.seed.device_words(self.dev).data_ptr(), self.seed.capacity,
                lay.frontier(self.base, slot, r), lay.partials(self.base, slot, r), lay.flag(self.base, slot, r), e,
                _lib.HTH_SLICE_ACCUMULATE, self.ws.data_ptr(), self.ws.numel(), st))
            if r != 0:
                return None
            _lib.check(L.hth_hash_merge_ex(
                p.output_bytes, plan.n_bytes, plan.level, lay.frontier(self.base, slot, 0), plan.n_frontier,
                lay.partials(self.base, slot), plan.n_slices, self.seed.device_words(self.dev).data_ptr(),
                self.seed.capacity, self.out[slot].data_ptr(), lay.flag(self.base, slot), e,
                lay.consumed(self.base, slot), self.timeout_ns, self.status_t.data_ptr(), self.mtmp.data_ptr(),
                self.mtmp.numel(), st))
            return self.out[slot]

    def check(self):
        """Synchronize; raise if a wait on this rank timed out."""
        import torch

        torch.cuda.synchronize(self.dev)
        if int(self.status_t.item()):
            raise RuntimeError(f"rank {self.rank}: a peer flag wait timed out; digests are invalid")


def hash_string_emulated(full, plan: SlicePlan, seed: SeedBuffer, epoch: int = 1, state=None, mark=None):
    """The FlagExchange protocol with every rank's slice run by ONE process on
    ONE device, one after another on one stream (the merge's flag wait is
    then satisfied before it starts: no kernel ever waits on a concurrently
    running one).  ``full``: the whole string on the device.  Exercises the
    same kernels, flags, slot reuse and partial re-zeroing as the multi-GPU
    path; used by the tests and the bench's single-GPU exchange cost.
    Returns (digest device tensor, state) -- pass state back for the next
    epoch (which must be the previous one + 1).  ``mark(tag)``, if given, is
    called before each launch ("slice<r>", "merge") and after the last
    ("end"), e.g. to record CUDA events."""
    import torch

    p = plan.params
    lay = _SlotLayout(plan)
    dev = full.device
    if state is None:
        k = lay.k
        wsz = ctypes.c_uint64()
        _lib.check(_lib.lib().hth_workspace_size_slice(p.output_bytes, plan.n_bytes, ctypes.byref(wsz)))
        state = {"buf": torch.zeros(lay.words, dtype=torch.int64, device=dev),
                 "ws": torch.zeros(max(wsz.value, 256), dtype=torch.uint8, device=dev),
                 "out": torch.zeros((2, k), dtype=torch.int64, device=dev),
                 "tmp": torch.empty(2 * (plan.n_frontier // 8 + 8) * 8 * k * 8, dtype=torch.uint8, device=dev),
                 "status": torch.zeros(1, dtype=torch.int32, device=dev)}
    base = state["buf"].data_ptr()
    L = _lib.lib()
    slot = (epoch - 1) & 1
    with torch.cuda.device(dev):
        st = torch.cuda.current_stream(dev).cuda_stream
        for r in range(plan.n_slices):
            b0, _ = plan.byte_range(r)
            if mark:
                mark(f"slice{r}")
            if r and epoch > 2:
                _lib.check(L.hth_wait_flag(lay.consumed(base, slot), epoch - 2, 10 ** 10,
                                           state["status"].data_ptr(), st))
            _lib.check(L.hth_hash_slice_ex(
                p.output_bytes, full.data_ptr() + b0, plan.n_bytes, plan.bounds[r], plan.bounds[r + 1], plan.level,
                seed.fold, seed.device_words(dev).data_ptr(), seed.capacity, lay.frontier(base, slot, r),
                lay.partials(base, slot, r), lay.flag(base, slot, r), epoch, _lib.HTH_SLICE_ACCUMULATE,
                state["ws"].data_ptr(), state["ws"].numel(), st))
        if mark:
            mark("merge")
        _lib.check(L.hth_hash_merge_ex(
            p.output_bytes, plan.n_bytes, plan.level, lay.frontier(base, slot, 0), plan.n_frontier,
            lay.partials(base, slot), plan.n_slices, seed.device_words(dev).data_ptr(), seed.capacity,
            state["out"][slot].data_ptr(), lay.flag(base, slot), epoch, lay.consumed(base, slot), 10 ** 10,
            state["status"].data_ptr(), state["tmp"].data_ptr(), state["tmp"].numel(), st))
        if mark:
            mark("end")
    return state["out"][slot], state
