"""Multi-GPU plumbing of the update phase: ZeRO-3 subgroup sharding and the
gradient exchange that feeds each rank's engine.

* shard(): contiguous subgroup blocks, the remainder spread over the first
  ranks — the reference's worker partition (harness.hpp:118-126).
* reduce_grads_to_owners(): sums every rank's 16-bit gradient contribution of
  each subgroup onto the rank that owns it. Even shards use one
  reduce_scatter over the flat, rank-contiguous gradient space; uneven shards
  (e.g. 690 subgroups over 8 ranks) use one reduce per subgroup to its owner
  (SURVEY §8e). Backend: NCCL over NVLink on GPUs, gloo on CPU (tests).
  The output buffers are what a rank binds into its engine with
  OffloadWorker.bind_grad_buffer (no copy).
* PeerGradients: the fused alternative — no collective on the data path.
  Every rank writes its contribution into one flat device buffer shared with
  the other ranks over CUDA IPC (NVLink peer mappings); the owner of a
  subgroup binds the world's slices of it with
  OffloadWorker.bind_grad_sources, and the update kernel sums them (fp32, in
  rank order, rounded once) while it streams the optimizer state.
"""
from __future__ import annotations

from typing import Dict, List, Sequence, Tuple


def shard(M: int, world: int, rank: int) -> Tuple[int, int]:
    """(first subgroup, count) owned by `rank` of `world` over M subgroups."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, rem = divmod(M, world)
    begin = rank * base + min(rank, rem)
    return begin, base + (1 if rank < rem else 0)


def owner_of(sg: int, M: int, world: int) -> int:
    for r in range(world):
        b, c = shard(M, world, r)
        if b <= sg < b + c:
            return r
    raise ValueError(f"subgroup {sg} out of range")


def reduce_grads_to_owners(local: Sequence, sizes: Sequence[int], world: int, rank: int, group=None) -> Dict[int, object]:
    """local[sg]: this rank's 16-bit (float16/bfloat16 torch tensor) gradient
    contribution for every subgroup sg. Returns {sg: summed gradient} for the
    subgroups this rank owns. The collectives are ordered on torch's current
    stream; the engine orders every run_update after its producer stream
    (OffloadWorker.set_producer_stream, default: the legacy default stream),
    so binding the results needs no host synchronisation when they are
    produced on that stream."""
    import torch
    import torch.distributed as dist

    M = len(sizes)
    if len(local) != M:
        raise ValueError("one local gradient per subgroup expected")
    begin, count = shard(M, world, rank)
    even = M % world == 0 and len(set(sizes)) == 1
    out: Dict[int, object] = {}
    if world == 1:
        return {sg: local[sg] for sg in range(M)}
    if even:
        flat = torch.cat([t.reshape(-1) for t in local])
        mine = torch.empty(count * sizes[0], dtype=flat.dtype, device=flat.device)
        dist.reduce_scatter_tensor(mine, flat, op=dist.ReduceOp.SUM, group=group)
        for k in range(count):
            out[begin + k] = mine[k * sizes[0]:(k + 1) * sizes[0]]
        return out
    for sg in range(M):
        dst = owner_of(sg, M, world)
        t = local[sg].clone() if dst == rank else local[sg]
        dist.reduce(t, dst=dst, op=dist.ReduceOp.SUM, group=group)
        if dst == rank:
            out[sg] = t
    return out


def parity_contribution(full_grad16, world: int, rank: int):
    """The rank-disjoint parity configuration: rank r keeps the
    reference gradient on elements i % world == r and exact zeros elsewhere,
    so the cross-rank sum reproduces the reference gradient regardless of the
    collective's reduction order."""
    import torch
    mask = (torch.arange(full_grad16.numel(), device=full_grad16.device) % world) == rank
    return torch.where(mask, full_grad16, torch.zeros_like(full_grad16))


def owned_ids(M: int, world: int, rank: int) -> List[int]:
    b, c = shard(M, world, rank)
    return list(range(b, b + c))


def contribution_layout(sizes: Sequence[int], world: int, window: int = 0) -> Tuple[List[int], int]:
    """(element offset of each subgroup's contribution, total elements) in a
    rank's PeerGradients buffer. window == 0: one 8-element-aligned slice per
    subgroup. window > 0: rolling buckets, subgroup k of owner o's shard in
    slot (k % window) * world + o, each slot max(sizes) rounded up to 8."""
    offsets: List[int] = []
    if window > 0:
        M = len(sizes)
        slot = (max(sizes) + 7) // 8 * 8
        for sg in range(M):
            o = owner_of(sg, M, world)
            k = sg - shard(M, world, o)[0]
            offsets.append(((k % window) * world + o) * slot)
        return offsets, window * world * slot
    off = 0
    for n in sizes:
        offsets.append(off)
        off += (n + 7) // 8 * 8
    return offsets, off


class _DeviceArray:
    """__cuda_array_interface__ view of a raw device range (torch.as_tensor)."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


class PeerGradients:
    """One flat 16-bit gradient buffer per rank covering every subgroup,
    mapped by every other rank over CUDA IPC.

    local(sg) is this rank's contribution to subgroup sg (a torch view to fill
    in backward); sources(sg) are the device pointers of all ranks'
    contributions in rank order, for OffloadWorker.bind_grad_sources on the
    owner. Subgroup slices start on 16-byte boundaries so the update kernel
    keeps its 128-bit loads. Synchronisation is the caller's: every rank's
    writes must be complete (stream synchronised + barrier) before an owner's
    run_update reads them, and every owner's update must be done (barrier)
    before a rank overwrites its buffer."""

    def __init__(self, sizes: Sequence[int], world: int, rank: int, device: int = 0, dtype: str = "f16",
                 group=None, window: int = 0):
        """window > 0: rolling buckets instead of one slice per subgroup. The
        backward emits gradients bucket by bucket and each bucket is consumed
        before the buffer is reused, so a rank only ever holds `window`
        subgroups per owner: subgroup k of owner o's shard lives in slot
        (k % window) * world + o (window x world slots of max(sizes)). The
        bytes an owner reads per subgroup are the same; device memory drops
        from 2 B x every param to 2 B x window x world x max(sizes)."""
        import torch.distributed as dist

        from . import tierflow as tf
        if dtype not in ("f16", "bf16"):
            raise ValueError("dtype must be f16 or bf16")
        self._tf, self.device, self.world, self.rank = tf, device, world, rank
        self.sizes = list(sizes)
        self.dtype = dtype
        self.window = window
        self.offsets, off = contribution_layout(self.sizes, world, window)
        self.total = max(off, 8)
        self._local = tf.device_alloc(device, 2 * self.total)
        self._opened: List[int] = []
        self.bases: List[int] = []
        try:
            handle = tf.ipc_get_handle(device, self._local)
            handles: List[object] = [None] * world
            if world > 1:
                dist.all_gather_object(handles, handle, group=group)
            else:
                handles = [handle]
            for r, h in enumerate(handles):
                if r == rank:
                    self.bases.append(self._local)
                else:
                    ptr = tf.ipc_open_handle(device, h)
                    self._opened.append(ptr)
                    self.bases.append(ptr)
        except BaseException:
            self.close()
            raise

    def local(self, sg: int):
        import torch
        dt = torch.float16 if self.dtype == "f16" else torch.bfloat16
        arr = _DeviceArray(self._local + 2 * self.offsets[sg], self.sizes[sg], "<i2")
        return torch.as_tensor(arr, device=f"cuda:{self.device}").view(dt)

    def slot_view(self, slot: int, count: int = 1):
        """window > 0: `count` consecutive bucket slots of this rank's buffer
        (a flat 16-bit torch view), e.g. to fill them in backward."""
        import torch
        if self.window <= 0:
            raise ValueError("slot_view needs a windowed PeerGradients")
        per = (max(self.sizes) + 7) // 8 * 8
        if not (0 <= slot and slot + count <= self.window * self.world):
            raise ValueError("bucket slot out of range")
        dt = torch.float16 if self.dtype == "f16" else torch.bfloat16
        arr = _DeviceArray(self._local + 2 * slot * per, count * per, "<i2")
        return torch.as_tensor(arr, device=f"cuda:{self.device}").view(dt)

    def sources(self, sg: int) -> List[int]:
        return [b + 2 * self.offsets[sg] for b in self.bases]

    def bind(self, worker, owned: Sequence[int]) -> None:
        """Bind every owned subgroup of `worker` to the world's contributions."""
        for sg in owned:
            worker.bind_grad_sources(sg, self.sources(sg))

    def close(self) -> None:
        for ptr in self._opened:
            self._tf.ipc_close_handle(self.device, ptr)
        self._opened = []
        if self._local:
            self._tf.device_free(self.device, self._local)
            self._local = 0

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
