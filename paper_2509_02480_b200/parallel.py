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
    subgroups this rank owns."""
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
