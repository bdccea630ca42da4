"""World-size-2 gloo runs of the multi-GPU host logic (CPU): contiguous
ZeRO-3 sharding (harness.hpp:118-126) and the gradient exchange in the
rank-disjoint parity configuration. The summed gradients, fed to
the Adam oracle on the owning rank, give the single-process oracle's bits."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2509_02480_b200 import parallel


def test_shard_matches_reference_partition():
    for M in range(1, 40):
        for world in range(1, 9):
            covered = []
            for r in range(world):
                b, c = parallel.shard(M, world, r)
                base, rem = divmod(M, world)
                assert b == r * base + min(r, rem) and c == base + (r < rem)
                covered += list(range(b, b + c))
            assert covered == list(range(M))
            assert all(parallel.owner_of(sg, M, world) == next(r for r in range(world)
                       if sg in parallel.owned_ids(M, world, r)) for sg in range(M))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, sizes, seed, result_q):
    import torch.distributed as dist

    import oracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        local = []
        for sg, n in enumerate(sizes):
            full = torch.from_numpy(oracle.synthetic_grads(n, seed, sg, 0).view(np.float16).copy())
            local.append(parallel.parity_contribution(full, world, rank))
        mine = parallel.reduce_grads_to_owners(local, sizes, world, rank)
        res = {}
        for sg, g in mine.items():
            g16 = g.numpy().view(np.uint16)
            n = sizes[sg]
            p0 = oracle.synthetic_params(n, seed, sg)
            p, m, v, p16, _ = oracle.adam_fused(p0, np.zeros(n, np.float32), np.zeros(n, np.float32), g16, 0, 0, 1)
            res[sg] = (g16.copy(), np.concatenate([p, m, v]).view(np.uint32).copy(), p16.copy())
        result_q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,sizes", [(2, [4096] * 4), (2, [4096, 4096, 4096, 1000, 777]),
                                         (3, [4096, 4096, 1000, 777, 3000]), (4, [2048] * 8)])
def test_gradient_exchange_parity(world, sizes):
    """World 2-4 over gloo: even shards (one reduce_scatter) and uneven ones
    (one reduce per subgroup to its owner, as C4's 86/87 split at N=8)."""
    import oracle
    seed = 9
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, sizes, seed, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(world):
        rank, res = q.get(timeout=120)
        for sg, v in res.items():
            assert parallel.owner_of(sg, len(sizes), world) == rank
            got[sg] = v
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    assert sorted(got) == list(range(len(sizes)))
    for sg, n in enumerate(sizes):
        want_g = oracle.synthetic_grads(n, seed, sg, 0)
        g16, pmv, p16 = got[sg]
        # identical up to the sign of zero (-0 + +0 = +0 in the sum)
        assert np.array_equal(g16 & 0x7FFF, want_g & 0x7FFF)
        assert np.array_equal(np.where(g16 == 0x8000, 0, g16), np.where(want_g == 0x8000, 0, want_g))
        p0 = oracle.synthetic_params(n, seed, sg)
        p, m, v, wp16, _ = oracle.adam_fused(p0, np.zeros(n, np.float32), np.zeros(n, np.float32), want_g, 0, 0, 1)
        assert np.array_equal(pmv, np.concatenate([p, m, v]).view(np.uint32))  # bit-exact state
        assert np.array_equal(p16, wp16)
