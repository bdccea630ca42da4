"""Fused data-parallel reduce + update: every rank's 16-bit
gradient contribution lives in its own HBM, mapped by the other ranks over
CUDA IPC (parallel.PeerGradients); the owner's engine binds the world's
slices with bind_grad_sources and its update kernel sums them (fp32, in rank
order, rounded once) while streaming P/m/v. No collective on the data path.

The world-2 case runs two processes on one GPU (IPC between processes on the
same device maps exactly as over NVLink, without peer hops). Expected bits
come from the oracle: sum the contributions in rank order in fp32, narrow
once, then the reference Adam."""
import os
import socket

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

SEED = 31


def _contribution(n, rank, sg, it, kind=0):
    return oracle.synthetic_grads(n, SEED + 100 * rank, sg, it, kind=kind)


def _expected(sizes, world, iters, kind=0, wd=0.0):
    out = {}
    for sg, n in enumerate(sizes):
        p = oracle.synthetic_params(n, SEED, sg)
        m = np.zeros(n, np.float32)
        v = np.zeros(n, np.float32)
        p16 = None
        for it in range(iters):
            acc = np.full(n, -0.0, np.float32)  # the in-order sum starts at source 0
            for r in range(world):
                acc = (acc + oracle.widen16(_contribution(n, r, sg, it, kind), kind)).astype(np.float32)
            g16, _ = oracle.narrow16(acc, kind)
            p, m, v, p16, _ = oracle.adam_fused(p, m, v, g16, kind, kind, it + 1, weight_decay=wd)
        out[sg] = (np.concatenate([p, m, v]).view(np.uint32), p16)
    return out


def _engine(tf, owned, sizes, lock_dir, kind=0, wd=0.0, pool=3, device=0):
    trace = tf.EventTrace()
    tiers = [tf.Tier(tf.TierSpec(0, tf.TierKind.host_dram, "dram", 20e9, 20e9))]
    w = tf.OffloadWorker(0, tiers, tf.ScheduleOptions(pool_slots=pool, lock_dir=lock_dir), tf.AdamHyper(weight_decay=wd),
                         trace, tf.DeviceOptions(device, kind, kind, 2))
    for sg in owned:
        w.add_subgroup(sg, sizes[sg])
    w.init_and_flush_all(SEED)
    return w, tiers


def _rank_main(rank, world, port, sizes, iters, lock_dir, q, distinct=False, window=0):
    import torch
    import torch.distributed as dist

    from paper_2509_02480_b200 import parallel, tierflow as tf
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dev = rank if distinct else 0  # distinct: one GPU per rank, peers mapped over NVLink / P2P
        torch.cuda.set_device(dev)
        owned = parallel.owned_ids(len(sizes), world, rank)
        w, _ = _engine(tf, owned, sizes, lock_dir, device=dev)
        with parallel.PeerGradients(sizes, world, rank, device=dev, window=window) as pg:
            pg.bind(w, owned)
            for it in range(iters):
                for sg, n in enumerate(sizes):  # "backward": this rank's contribution to every subgroup
                    g = torch.from_numpy(_contribution(n, rank, sg, it).view(np.int16))
                    pg.local(sg).view(torch.int16).copy_(g.to(f"cuda:{dev}"))
                torch.cuda.synchronize()
                dist.barrier()  # every contribution written before any owner reads it
                w.run_update(it)
                dist.barrier()  # every owner done before the buffers are overwritten
            res = {sg: (w.read_current_state(sg).view(np.uint32).copy(), w.read_params16(sg).copy()) for sg in owned}
        w.close()
        q.put((rank, res, None))
    except BaseException as e:  # noqa: BLE001 - surfaced in the parent
        q.put((rank, {}, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.parametrize("sizes,distinct,window", [
    ([50_000, 50_000, 50_000, 50_000], False, 0),
    ([70_001, 4_097, 33_333], False, 0),
    ([50_000, 50_000, 50_000, 50_000], False, 2),  # rolling-bucket layout (the bench's C3 exchange)
    pytest.param([50_000, 50_000, 50_000, 50_000], True, 0,
                 marks=pytest.mark.skipif(_gpus() < 2, reason="needs two GPUs (ranks on distinct devices)")),
    pytest.param([70_001, 4_097, 33_333], True, 2,
                 marks=pytest.mark.skipif(_gpus() < 2, reason="needs two GPUs (ranks on distinct devices)")),
])
def test_ipc_fused_exchange_world2(tf, cuda, tmp_path, sizes, distinct, window):
    """world 2; distinct=True puts each rank on its own GPU so every peer
    contribution crosses NVLink / P2P (skipped on a one-GPU box)."""
    import torch.multiprocessing as mp
    world, iters = 2, 2
    lock_dir = tmp_path / "locks"
    lock_dir.mkdir()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, sizes, iters, str(lock_dir), q, distinct, window))
             for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    try:
        for _ in range(world):
            rank, res, err = q.get(timeout=300)
            assert err is None, f"rank {rank}: {err}"
            got.update(res)
    finally:
        for p in procs:
            p.join(60)
    assert all(p.exitcode == 0 for p in procs)
    want = _expected(sizes, world, iters)
    assert sorted(got) == list(range(len(sizes)))
    for sg in range(len(sizes)):
        assert np.array_equal(got[sg][0], want[sg][0]), f"subgroup {sg} state"
        assert np.array_equal(got[sg][1], want[sg][1]), f"subgroup {sg} params16"


@pytest.mark.parametrize("nsrc,kind", [(1, 0), (3, 0), (8, 1)])
def test_engine_multi_source_binding(tf, cuda, lock_dir, nsrc, kind):
    """In-process: n device buffers bound as one subgroup's sources; the
    engine's update equals the oracle on the in-order fp32 sum."""
    import torch
    sizes = [40_000, 12_345]
    w, _ = _engine(tf, [0, 1], sizes, lock_dir, kind=kind, wd=0.01)
    bufs = {sg: [torch.from_numpy(_contribution(n, r, sg, 0, kind).view(np.int16)).cuda() for r in range(nsrc)]
            for sg, n in enumerate(sizes)}
    for sg in range(2):
        w.bind_grad_sources(sg, [b.data_ptr() for b in bufs[sg]])
    w.run_update(0)
    want = _expected(sizes, nsrc, 1, kind=kind, wd=0.01)
    for sg in range(2):
        assert np.array_equal(w.read_current_state(sg).view(np.uint32), want[sg][0])
        assert np.array_equal(w.read_params16(sg), want[sg][1])
    w.close()


def test_sum_overflow_rejected_before_mutation(tf, cuda, lock_dir):
    """Finite sources whose sum overflows f16: the whole-phase pre-check sees
    the reduced gradient, raises GradientOverflowError, and no state moves."""
    import torch
    n = 10_000
    w, _ = _engine(tf, [0], [n], lock_dir)
    before = w.read_current_state(0).copy()
    big = torch.full((n,), 40000.0, dtype=torch.float16, device=cuda)
    w.bind_grad_sources(0, [big.data_ptr(), big.data_ptr()])
    assert not w.gradients_finite()
    with pytest.raises(tf.GradientOverflowError):
        w.run_update(0)
    assert np.array_equal(w.read_current_state(0), before)
    # rebinding a single buffer clears the sources
    ok = torch.full((n,), 0.5, dtype=torch.float16, device=cuda)
    w.bind_grad_buffer(0, ok.data_ptr())
    assert w.gradients_finite()
    w.close()


def test_bind_sources_rejected_in_baseline_flow(tf, cuda, lock_dir):
    trace = tf.EventTrace()
    tiers = [tf.Tier(tf.TierSpec(0, tf.TierKind.host_dram, "dram", 20e9, 20e9))]
    w = tf.OffloadWorker(0, tiers, tf.ScheduleOptions(pool_slots=3, lock_dir=lock_dir, skip_gradients=False),
                         tf.AdamHyper(), trace, tf.DeviceOptions(0, 0, 0, 2))
    w.add_subgroup(0, 1000)
    w.init_and_flush_all(SEED)
    import torch
    b = torch.zeros(1000, dtype=torch.float16, device=cuda)
    with pytest.raises(tf.ConfigError):
        w.bind_grad_sources(0, [b.data_ptr(), b.data_ptr()])
    with pytest.raises(tf.ConfigError):
        w.bind_grad_sources(0, [b.data_ptr()] * 9)
    w.close()
