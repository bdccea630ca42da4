"""The B200 update engine against the reference engine (golden fixtures from
the unmodified reference, tests/golden/make_golden.py) and the oracle (-m gpu).

Bit-exact: cache-hit counts and ids, per-tier prefetch order, per-tier flush
sets, flush allocations, retained counts and the final P/m/v bits. The
scenarios mirror the reference's test_scheduler.cpp."""
import ast
import hashlib
import threading
import time

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def make_engine(tf, tiers_cfg, params, *, pool_slots=4, cache_slots=-1, ratio=None, seed=42, lock_dir="",
                wd=0.0, device_buffers=3, grad_dtype=0, param_dtype=0, deadlock=30.0, pad_ns=0, caching=True,
                multi_path=True, hbm=1, lock_device=0, host_grads=False):
    trace = tf.EventTrace()
    tiers = [tf.Tier(tf.TierSpec(i, *cfg, lock_device=lock_device)) for i, cfg in enumerate(tiers_cfg)]
    opt = tf.ScheduleOptions(pool_slots=pool_slots, cache_slots=cache_slots, lock_dir=lock_dir,
                             deadlock_timeout_s=deadlock, update_pad_ns=pad_ns, enable_caching=caching,
                             multi_path=multi_path)
    w = tf.OffloadWorker(0, tiers, opt, tf.AdamHyper(weight_decay=wd), trace,
                         tf.DeviceOptions(0, grad_dtype, param_dtype, device_buffers, 0, 1, hbm, host_grads=host_grads))
    if ratio is not None:
        w.set_fixed_ratio(ratio)
    for i, n in enumerate(params):
        w.add_subgroup(i, n)
    w.init_and_flush_all(seed)
    return w, trace, tiers


def mem(rate_r, rate_w):
    return (2, "mem", rate_r, rate_w)


def run_golden(tf, golden, run, lock_dir, device_buffers=3, hbm=1, host_slots=None, host_grads=False):
    cfg = golden[f"run_{run}_config"]
    M, nt, pool, cache, seed, iters, accum, skip = (int(x) for x in cfg)
    if hbm == 2:  # HBM cache: the reference's C on HBM, `host_slots` pool slots all streaming
        cache = tf.retention_capacity(True, pool, cache, M)
        pool = host_slots
    params = golden[f"run_{run}_params"].tolist()
    rates = {"hits": [(500e6, 500e6), (250e6, 250e6)], "ragged": [(300e6, 300e6), (200e6, 200e6), (100e6, 100e6)],
             "skip": [(400e6, 400e6), (200e6, 200e6)], "desk10": [(4000e6, 4000e6), (2000e6, 2000e6)]}[run]
    w, trace, tiers = make_engine(tf, [mem(*r) for r in rates], params, pool_slots=pool, cache_slots=cache,
                                  ratio=golden[f"run_{run}_ratio"].tolist(), seed=seed, lock_dir=lock_dir,
                                  wd=float(golden[f"run_{run}_wd"][0]), device_buffers=device_buffers, hbm=hbm,
                                  host_grads=host_grads)
    stats, seqs = [], []
    for it in range(iters):
        w.run_backward_sim(it, tf.SyntheticGradSource(seed), accum)
        if (skip >> it) & 1:
            stats.append(None)
            seqs.append({"hits": [], "prefetch": [[] for _ in range(nt)], "flush": [[] for _ in range(nt)]})
            continue
        mark = trace.size()
        st = w.run_update(it)
        ev = [(int(e.kind), e.subgroup_id, e.tier_id, e.bytes) for e in trace.snapshot(mark)]
        seqs.append(oracle.phase_sequences(ev, 0, len(ev), nt))
        stats.append(st)
    return w, trace, stats, seqs, params, iters


@pytest.mark.parametrize("run,hbm,host_slots", [("hits", 1, None), ("ragged", 1, None), ("skip", 1, None),
                                                ("hits", 2, 3), ("ragged", 2, 3), ("skip", 2, 4)])
def test_sequences_and_state_match_reference_engine(tf, cuda, golden, lock_dir, run, hbm, host_slots):
    """hbm=2 (HBM cache mode): the reference's retention capacity held in HBM
    with only `host_slots` pinned slots: same sequences, counts and bits."""
    w, trace, stats, seqs, params, iters = run_golden(tf, golden, run, lock_dir, hbm=hbm, host_slots=host_slots)
    want_seqs = [ast.literal_eval(s) for s in golden[f"run_{run}_seqs"]]
    for it in range(iters):
        assert seqs[it] == want_seqs[it], f"iteration {it}"
        if stats[it] is None:
            continue
        assert stats[it].cache_hits == golden[f"run_{run}_hits"][it]
        assert stats[it].retained == golden[f"run_{run}_retained"][it]
        assert stats[it].flush_allocation == golden[f"run_{run}_alloc"][it].tolist()
        assert stats[it].downscale_overflows == golden[f"run_{run}_overflows"][it]
        assert stats[it].params_updated == sum(params)
    if run == "hits":
        assert [s.cache_hits for s in stats] == [0, 4, 4, 4]
        for i in range(len(params)):
            d = hashlib.sha256(w.read_current_state(i).tobytes()).hexdigest()
            assert d == golden["run_hits_digest"][i], f"subgroup {i}"
    else:
        ref = golden[f"run_{run}_states"]
        off = 0
        for i, n in enumerate(params):
            got = w.read_current_state(i)
            assert np.array_equal(got.view(np.uint32), ref[off:off + 3 * n].view(np.uint32)), f"subgroup {i}"
            # device working params = RNE(P) of the final state
            assert np.array_equal(w.read_params16(i), oracle.f32_to_f16(got[:n]))
            off += 3 * n
    w.close()


@pytest.mark.parametrize("hbm,host_slots,host_grads", [(1, None, False), (2, 3, False), (2, 3, True)])
def test_ten_step_contract_on_the_desk_shape(tf, cuda, golden, lock_dir, hbm, host_slots, host_grads):
    """north_star: results after 10 steps. The reference engine on its desk
    shape (configs/desk.json: 24 subgroups x 2,796,202, P % 4 = 2), AdamW
    (wd 0.01), C = 4, 12 iterations with iteration 5 skipped (11 applied):
    every phase's cache hits, per-tier fetch order, flush sets and allocation,
    then the final P/m/v and working params of every subgroup, bit for bit."""
    w, trace, stats, seqs, params, iters = run_golden(tf, golden, "desk10", lock_dir, hbm=hbm, host_slots=host_slots,
                                                      host_grads=host_grads)
    want_seqs = [ast.literal_eval(s) for s in golden["run_desk10_seqs"]]
    assert iters == 12 and sum(st is not None for st in stats) == 11
    for it in range(iters):
        assert seqs[it] == want_seqs[it], f"iteration {it}"
        if stats[it] is None:
            continue
        assert stats[it].cache_hits == golden["run_desk10_hits"][it]
        assert stats[it].retained == golden["run_desk10_retained"][it]
        assert stats[it].flush_allocation == golden["run_desk10_alloc"][it].tolist()
        assert stats[it].downscale_overflows == golden["run_desk10_overflows"][it]
    # after the skipped iteration the direction repeats, so the hits of iteration 6 come last in its order
    assert [s.cache_hits for s in stats if s is not None] == [0] + [4] * 10
    for i, n in enumerate(params):
        got = w.read_current_state(i)
        assert hashlib.sha256(got.tobytes()).hexdigest() == golden["run_desk10_digest"][i], f"subgroup {i}"
        assert np.array_equal(w.read_params16(i), oracle.f32_to_f16(got[:n]))
    w.close()


@pytest.mark.parametrize("run,hbm,host_slots", [("ragged", 1, None), ("skip", 2, 4), ("hits", 2, 3)])
def test_host_resident_grads_match_reference_engine(tf, cuda, golden, lock_dir, run, hbm, host_slots):
    """DeviceOptions.host_grads: the 16-bit gradients and working params live
    in pinned host blocks and stream with the state (no HBM arenas for the
    shard). Same sequences and bits as the reference; the PCIe byte count
    carries the 2 B/param each way; the working params read back from host."""
    w, trace, stats, seqs, params, iters = run_golden(tf, golden, run, lock_dir, hbm=hbm, host_slots=host_slots,
                                                      host_grads=True)
    want_seqs = [ast.literal_eval(s) for s in golden[f"run_{run}_seqs"]]
    S = sum(params)
    for it in range(iters):
        assert seqs[it] == want_seqs[it], f"iteration {it}"
        if stats[it] is None:
            continue
        assert stats[it].cache_hits == golden[f"run_{run}_hits"][it]
        assert stats[it].flush_allocation == golden[f"run_{run}_alloc"][it].tolist()
        assert stats[it].h2d_bytes >= 2 * S and stats[it].d2h_bytes >= 2 * S
    for i, n in enumerate(params):
        got = w.read_current_state(i)
        if run == "hits":
            assert hashlib.sha256(got.tobytes()).hexdigest() == golden["run_hits_digest"][i]
        else:
            off = sum(3 * m for m in params[:i])
            assert np.array_equal(got.view(np.uint32), golden[f"run_{run}_states"][off:off + 3 * n].view(np.uint32))
        assert np.array_equal(w.read_params16(i), oracle.f32_to_f16(got[:n]))
    w.close()


def test_host_resident_grads_reject_a_nonfinite_phase(tf, cuda, lock_dir):
    """A gradient the caller writes into the host block (grad_buffer returns a
    pinned host pointer with host_grads): not counted by a producer, so the
    phase check stages it to the device; a poisoned one rejects the phase."""
    import ctypes
    n = 10_000
    w, trace, _ = make_engine(tf, [mem(800e6, 800e6)], [n] * 3, pool_slots=3, lock_dir=lock_dir, host_grads=True)
    w.run_backward_sim(0, tf.SyntheticGradSource(29))
    before = [w.read_current_state(i) for i in range(3)]
    host = np.ctypeslib.as_array((ctypes.c_uint16 * n).from_address(w.grad_buffer(1)))
    keep = host[77]
    host[77] = 0x7C00
    assert not w.gradients_finite()
    with pytest.raises(tf.GradientOverflowError):
        w.run_update(0)
    for i in range(3):
        assert np.array_equal(w.read_current_state(i), before[i])
    host[77] = keep
    st = w.run_update(1)
    assert st.cache_hits == 0 and st.params_updated == 3 * n
    p0 = oracle.synthetic_params(n, 42, 1)
    want = oracle.adam_fused(p0, np.zeros(n, np.float32), np.zeros(n, np.float32),
                             oracle.synthetic_grads(n, 29, 1, 0), 0, 0, 2)
    assert np.array_equal(w.read_current_state(1).view(np.uint32), np.concatenate(want[:3]).view(np.uint32))
    w.close()


@pytest.mark.parametrize("ring", [1, 2, 5])
def test_ring_depth_does_not_change_bits(tf, cuda, golden, lock_dir, ring):
    w, _, _, _, params, _ = run_golden(tf, golden, "ragged", lock_dir, device_buffers=ring)
    ref = golden["run_ragged_states"]
    off = 0
    for i, n in enumerate(params):
        assert np.array_equal(w.read_current_state(i).view(np.uint32), ref[off:off + 3 * n].view(np.uint32))
        off += 3 * n
    w.close()


def test_exactly_once_and_no_self_overlap(tf, cuda, lock_dir):
    w, trace, _ = make_engine(tf, [mem(250e6, 250e6), mem(125e6, 125e6)], [350_000] * 8, pool_slots=4,
                              lock_dir=lock_dir, pad_ns=8_000_000)
    w.run_backward_sim(0, tf.SyntheticGradSource(3))
    w.run_update(0)
    ev = trace.snapshot()
    iv = {}
    for kind_s, kind_e in [("prefetch_start", "prefetch_end"), ("update_start", "update_end"),
                           ("flush_start", "flush_end")]:
        opened, out = {}, []
        for e in ev:
            if e.kind == tf.EventKind[kind_s]:
                opened[e.subgroup_id] = e.timestamp_ns
            elif e.kind == tf.EventKind[kind_e]:
                out.append((opened.pop(e.subgroup_id), e.timestamp_ns, e.subgroup_id))
        assert not opened
        iv[kind_s] = out
    ups = iv["update_start"]
    assert sorted(u[2] for u in ups) == list(range(8))  # exactly once
    ov = lambda a, b: max(a[0], b[0]) < min(a[1], b[1])
    for u in ups:
        for x in iv["prefetch_start"] + iv["flush_start"]:
            if x[2] == u[2]:
                assert not ov(u, x)
    three = any(ov(u, p) and ov(u, f) and max(u[0], p[0], f[0]) < min(u[1], p[1], f[1])
                for u in ups for p in iv["prefetch_start"] for f in iv["flush_start"])
    assert three, "prefetch, update and flush never simultaneously in flight"
    w.close()


def test_nonfinite_gradient_rejects_phase_without_mutation(tf, cuda, lock_dir):
    import torch
    n = 10_000
    w, trace, _ = make_engine(tf, [mem(800e6, 800e6)], [n] * 3, pool_slots=3, lock_dir=lock_dir)
    w.run_backward_sim(0, tf.SyntheticGradSource(29))
    before = [w.read_current_state(i) for i in range(3)]
    g16 = oracle.synthetic_grads(n, 29, 1, 0)
    g16[77] = 0x7C00
    bad = torch.from_numpy(g16.view(np.int16)).cuda()
    w.bind_grad_buffer(1, bad.data_ptr())
    assert not w.gradients_finite()
    with pytest.raises(tf.GradientOverflowError):
        w.run_update(0)
    for i in range(3):
        assert np.array_equal(w.read_current_state(i), before[i])
    # the harness skips the step; iteration 1 proceeds (Adam t = 2, parity key 1)
    g16[77] = 0
    good = torch.from_numpy(g16.view(np.int16)).cuda()
    w.bind_grad_buffer(1, good.data_ptr())
    assert w.gradients_finite()
    st = w.run_update(1)
    assert st.params_updated == 3 * n
    assert st.cache_hits == 0  # the rejected phase's fetches were rolled back to their tier
    p0 = oracle.synthetic_params(n, 42, 1)
    want = oracle.adam_fused(p0, np.zeros(n, np.float32), np.zeros(n, np.float32), g16, 0, 0, 2)
    assert np.array_equal(w.read_current_state(1).view(np.uint32), np.concatenate(want[:3]).view(np.uint32))
    w.close()


def test_prefetch_of_retained_subgroup_is_cache_hit(tf, cuda, lock_dir):
    # test_scheduler.cpp:459-476
    w, trace, _ = make_engine(tf, [mem(800e6, 800e6)], [10_000] * 2, pool_slots=4, lock_dir=lock_dir)
    w.run_backward_sim(0, tf.SyntheticGradSource(23))
    w.run_update(0)
    assert w.meta(1).residency == tf.Residency.host_cached
    mark = trace.size()
    assert w.enqueue_prefetch(1) is None
    assert any(e.kind == tf.EventKind.cache_hit and e.subgroup_id == 1 for e in trace.snapshot(mark))
    w.close()


def test_never_enqueued_subgroup_fetched_on_demand(tf, cuda, lock_dir):
    # test_scheduler.cpp:522-535
    w, trace, _ = make_engine(tf, [mem(400e6, 400e6)], [20_000] * 2, pool_slots=3, lock_dir=lock_dir)
    assert w.meta(1).residency == tf.Residency.on_tier
    assert w.wait_host_resident(1) >= 0
    assert w.meta(1).residency == tf.Residency.host_cached
    assert any(e.kind == tf.EventKind.prefetch_end and e.subgroup_id == 1 for e in trace.snapshot())
    w.close()


def test_queued_flush_defers_until_lock_release(tf, cuda, lock_dir):
    # test_scheduler.cpp:409-435
    w, trace, _ = make_engine(tf, [mem(800e6, 800e6)], [20_000], pool_slots=3, lock_dir=lock_dir)
    w.enqueue_prefetch(0).get()
    guard = tf.acquire_tier_lock(lock_dir, 0, 99, trace)
    fl = w.enqueue_flush(0, 0)
    time.sleep(0.08)
    released = time.monotonic_ns()
    guard.release()
    fl.get()
    start = [e.timestamp_ns for e in trace.snapshot() if e.kind == tf.EventKind.flush_start and e.subgroup_id == 0]
    assert start and start[0] >= released
    w.close()


def test_flushes_to_distinct_tiers_overlap(tf, cuda, lock_dir):
    # test_scheduler.cpp:437-457
    w, trace, _ = make_engine(tf, [mem(150e6, 150e6), mem(150e6, 150e6)], [350_000] * 2, pool_slots=4,
                              lock_dir=lock_dir)
    for i in (0, 1):
        t = w.enqueue_prefetch(i)
        if t:
            t.get()
    mark = trace.size()
    f0, f1 = w.enqueue_flush(0, 0), w.enqueue_flush(1, 1)
    f0.get()
    f1.get()
    ev = trace.snapshot(mark)
    iv = {}
    for e in ev:
        if e.kind == tf.EventKind.flush_start:
            iv[e.subgroup_id] = [e.timestamp_ns, None, e.tier_id]
        elif e.kind == tf.EventKind.flush_end:
            iv[e.subgroup_id][1] = e.timestamp_ns
    a, b = iv[0], iv[1]
    assert a[2] != b[2] and max(a[0], b[0]) < min(a[1], b[1])
    w.close()


def test_tiers_on_one_device_share_the_semaphore(tf, cuda, lock_dir):
    """TierSpec.lock_device: two tiers keyed to one physical device take one
    semaphore, so their transfers serialise (contention control per device)."""
    w, trace, _ = make_engine(tf, [mem(150e6, 150e6), mem(150e6, 150e6)], [350_000] * 2, pool_slots=4,
                              lock_dir=lock_dir, lock_device=7)
    for i in (0, 1):
        t = w.enqueue_prefetch(i)
        if t:
            t.get()
    mark = trace.size()
    f0, f1 = w.enqueue_flush(0, 0), w.enqueue_flush(1, 1)
    f0.get()
    f1.get()
    iv = {}
    for e in trace.snapshot(mark):
        if e.kind == tf.EventKind.flush_start:
            iv[e.subgroup_id] = [e.timestamp_ns, None]
        elif e.kind == tf.EventKind.flush_end:
            iv[e.subgroup_id][1] = e.timestamp_ns
    a, b = sorted(iv.values())
    assert a[1] <= b[0]
    import os
    assert os.path.exists(os.path.join(lock_dir, "device_7.lock"))
    w.close()


def test_wedged_pipeline_trips_watchdog(tf, cuda, lock_dir):
    # test_scheduler.cpp:537-550
    w, trace, _ = make_engine(tf, [mem(800e6, 800e6)], [10_000], pool_slots=3, lock_dir=lock_dir, deadlock=0.4)
    w.run_backward_sim(0, tf.SyntheticGradSource(29))
    guard = tf.TierLockGuard(lock_dir, 0, 98, trace)
    with pytest.raises(tf.SchedulingBugError):
        w.run_update(0)
    guard.release()
    time.sleep(0.2)
    w.close()


def test_dram_and_directory_tiers_zero_copy_path(tf, cuda, lock_dir, tmp_path):
    """The B200 fast path: host_dram (block exchange) + local_dir (O_DIRECT
    into pinned slots), ragged sizes; end state equals the oracle bitwise and
    the on-disk files stay v1."""
    params = [100_003, 100_000, 64_001, 100_000, 99_999]
    tiers = [(3, "dram", 20e9, 20e9), (0, str(tmp_path / "nvme"), 3e9, 2e9)]
    w, trace, tier_objs = make_engine(tf, tiers, params, pool_slots=5, ratio=[2.0, 1.0], seed=11, lock_dir=lock_dir,
                                      wd=0.01)
    iters = 4
    held = []  # HBM-retained by the previous phase (C = 5 - 3): no H2D this phase
    for it in range(iters):
        w.run_backward_sim(it, tf.SyntheticGradSource(11), 1)
        st = w.run_update(it)
        assert st.params_updated == sum(params)
        assert st.h2d_bytes == 12 * (sum(params) - sum(params[i] for i in held)) and st.kernel_seconds > 0
        order = list(range(5)) if it % 2 == 0 else list(range(4, -1, -1))
        held = order[-2:]
    states, (order, hit, dest, origin) = oracle.run_engine_oracle(params, 11, iters, 5, -1, True, True, [2.0, 1.0],
                                                                  weight_decay=0.01)
    for i, n in enumerate(params):
        got = w.read_current_state(i)
        want = np.concatenate(states[i][:3])
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), f"subgroup {i}"
        assert np.array_equal(w.read_params16(i), states[i][3])
    on_disk = [i for i in range(len(params)) if w.meta(i).residency == tf.Residency.on_tier and w.meta(i).tier == 1]
    for i in on_disk:
        raw = (tmp_path / "nvme" / f"sg_{i:06d}.bin").read_bytes()
        assert raw[:4] == b"OPLM" and len(raw) == 32 + 12 * params[i]
    w.close()


def test_bf16_engine_matches_oracle(tf, cuda, lock_dir):
    params = [50_000, 33_333]
    w, _, _ = make_engine(tf, [mem(2e9, 2e9)], params, pool_slots=4, seed=3, lock_dir=lock_dir, grad_dtype=1,
                          param_dtype=1)
    for it in range(3):
        w.run_backward_sim(it, tf.SyntheticGradSource(3), 2)
        w.run_update(it)
    states, _ = oracle.run_engine_oracle(params, 3, 3, 4, -1, True, True, [1.0], accum_steps=2, grad_kind=1,
                                         out_kind=1)
    for i in range(2):
        assert np.array_equal(w.read_current_state(i).view(np.uint32),
                              np.concatenate(states[i][:3]).view(np.uint32))
        assert np.array_equal(w.read_params16(i), states[i][3])
    w.close()


def test_external_gradient_buffer_binding(tf, cuda, lock_dir):
    """A caller-owned device gradient buffer (e.g. a reduce-scatter output)."""
    import torch
    n = 40_000
    w, _, _ = make_engine(tf, [mem(2e9, 2e9)], [n], pool_slots=3, seed=8, lock_dir=lock_dir)
    g16 = oracle.synthetic_grads(n, 123, 0, 0)
    buf = torch.from_numpy(g16.view(np.int16)).cuda()
    w.bind_grad_buffer(0, buf.data_ptr())
    w.run_update(0)
    p0 = oracle.synthetic_params(n, 8, 0)
    want = oracle.adam_fused(p0, np.zeros(n, np.float32), np.zeros(n, np.float32), g16, 0, 0, 1)
    got = w.read_current_state(0)
    assert np.array_equal(got.view(np.uint32), np.concatenate(want[:3]).view(np.uint32))
    w.close()


@pytest.mark.parametrize("zero_copy,split", [(1, 1), (0, 2), (2, 1)])
def test_transfer_modes_bitwise(tf, cuda, lock_dir, tmp_path, zero_copy, split):
    """Zero-copy (kernel streams the pinned slot over PCIe) and split-D2H
    copy mode give the same bits as the oracle."""
    params = [100_000, 64_000, 99_996]
    trace = tf.EventTrace()
    tiers = [tf.Tier(tf.TierSpec(0, tf.TierKind.host_dram, "dram", 20e9, 20e9)),
             tf.Tier(tf.TierSpec(1, tf.TierKind.local_dir, str(tmp_path / "d"), 2e9, 2e9))]
    w = tf.OffloadWorker(0, tiers, tf.ScheduleOptions(pool_slots=5, lock_dir=lock_dir), tf.AdamHyper(), trace,
                         tf.DeviceOptions(0, 0, 0, 2, zero_copy, split))
    w.set_fixed_ratio([1.0, 1.0])
    for i, n in enumerate(params):
        w.add_subgroup(i, n)
    w.init_and_flush_all(17)
    for it in range(3):
        w.run_backward_sim(it, tf.SyntheticGradSource(17))
        w.run_update(it)
    states, _ = oracle.run_engine_oracle(params, 17, 3, 5, -1, True, True, [1.0, 1.0])
    for i in range(len(params)):
        assert np.array_equal(w.read_current_state(i).view(np.uint32), np.concatenate(states[i][:3]).view(np.uint32))
        assert np.array_equal(w.read_params16(i), states[i][3])
    tl = w.last_timeline()
    assert len(tl) == len(params) and all(s["k_end"] >= s["k_start"] for s in tl)
    w.close()


@pytest.mark.parametrize("zero_copy,skip", [(0, True), (2, True), (2, False), (0, False)])
def test_ring_reuse_under_slow_kernels(tf, cuda, lock_dir, tmp_path, zero_copy, skip):
    """Many more streaming subgroups than ring buffers, no retention, and a
    padded (slow) kernel: an H2D into a ring buffer must wait until the last
    kernel reading it is done (zero_copy=2 never recorded the
    buffer's release event). skip=False is the ZeRO-3 baseline flow, whose
    fp32 gradient segment shares the ring buffer's release."""
    params = [40_000 + 4 * i for i in range(10)]
    seed = 31
    trace = tf.EventTrace()
    tiers = [tf.Tier(tf.TierSpec(0, tf.TierKind.host_dram, "dram", 20e9, 20e9))]
    opt = tf.ScheduleOptions(pool_slots=8, cache_slots=0, lock_dir=lock_dir, enable_caching=False,
                             skip_gradients=skip, update_pad_ns=3_000_000)
    w = tf.OffloadWorker(0, tiers, opt, tf.AdamHyper(), trace, tf.DeviceOptions(0, 0, 0, 2, zero_copy, 1, 0))
    for i, n in enumerate(params):
        w.add_subgroup(i, n)
    w.init_and_flush_all(seed)
    for it in range(3):
        w.run_backward_sim(it, tf.SyntheticGradSource(seed))
        st = w.run_update(it)
        assert st.cache_hits == 0
    for sg, n in enumerate(params):
        p, m, v = oracle.synthetic_params(n, seed, sg), np.zeros(n, np.float32), np.zeros(n, np.float32)
        for it in range(3):
            p, m, v, p16, _ = oracle.adam_fused(p, m, v, oracle.synthetic_grads(n, seed, sg, it), 0, 0, it + 1)
        assert np.array_equal(w.read_current_state(sg).view(np.uint32), np.concatenate([p, m, v]).view(np.uint32)), sg
        assert np.array_equal(w.read_params16(sg), p16), sg
    w.close()


def _baseline_engine(tf, params, lock_dir, *, baseline, seed=1234, pool_slots=6):
    trace = tf.EventTrace()
    tiers = [tf.Tier(tf.TierSpec(0, tf.TierKind.mem_throttled, "m0", 300e6, 300e6)),
             tf.Tier(tf.TierSpec(1, tf.TierKind.mem_throttled, "m1", 150e6, 150e6))]
    opt = tf.ScheduleOptions(pool_slots=pool_slots, lock_dir=lock_dir, enable_caching=not baseline,
                             skip_gradients=not baseline, atomic_rw=not baseline, multi_path=not baseline)
    w = tf.OffloadWorker(0, tiers, opt, tf.AdamHyper(), trace, tf.DeviceOptions(0))
    for i, n in enumerate(params):
        w.add_subgroup(i, n)
    w.init_and_flush_all(seed)
    return w, trace, tiers


def test_zero3_baseline_flow_matches_reference(tf, cuda, golden, lock_dir):
    """skip_gradients=false: fp32 gradients flushed in backward (4 B/param) and
    fetched with the state (16 B/param) — reference scheduler.hpp:377-391,
    667-680; test_scheduler.cpp:357-390."""
    params = golden["run_baseline_params"].tolist()
    cfg = golden["run_baseline_config"]
    iters, accum, seed = int(cfg[5]), int(cfg[6]), int(cfg[4])
    w, trace, _ = _baseline_engine(tf, params, lock_dir, baseline=True, seed=seed)
    want_seqs = [ast.literal_eval(s) for s in golden["run_baseline_seqs"]]
    for it in range(iters):
        m0 = trace.size()
        w.run_backward_sim(it, tf.SyntheticGradSource(seed), accum)
        bw = sum(e.bytes for e in trace.snapshot(m0) if e.kind == tf.EventKind.flush_end)
        assert bw == golden["run_baseline_backward_bytes"][it] == 4 * sum(params)
        m1 = trace.size()
        st = w.run_update(it)
        ev = trace.snapshot(m1)
        fetched = sum(e.bytes for e in ev if e.kind == tf.EventKind.prefetch_end)
        assert fetched == golden["run_baseline_fetch_bytes"][it] == 16 * sum(params)
        seq = oracle.phase_sequences([(int(e.kind), e.subgroup_id, e.tier_id, e.bytes) for e in ev], 0, len(ev), 2)
        assert seq == want_seqs[it]
        assert st.cache_hits == 0 and st.flush_allocation == golden["run_baseline_alloc"][it].tolist()
    for i in range(len(params)):
        assert hashlib.sha256(w.read_current_state(i).tobytes()).hexdigest() == golden["run_baseline_digest"][i]
    w.close()


def test_engine_and_baseline_modes_bitwise_identical(tf, cuda, lock_dir):
    # acceptance criterion 4 / test_scheduler.cpp:329-355
    params = [30_000] * 6
    out = []
    for baseline in (False, True):
        w, _, _ = _baseline_engine(tf, params, lock_dir, baseline=baseline)
        for it in range(4):
            w.run_backward_sim(it, tf.SyntheticGradSource(1234), 2)
            w.run_update(it)
        out.append([w.read_current_state(i) for i in range(6)])
        w.close()
    for a, b in zip(*out):
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_engine_mode_backward_writes_nothing(tf, cuda, lock_dir):
    # acceptance criterion 6: backward-phase tier writes: engine 0, baseline 4*P*M
    P, M = 25_000, 5
    for baseline, want in ((False, 0), (True, 4 * P * M)):
        w, trace, _ = _baseline_engine(tf, [P] * M, lock_dir, baseline=baseline, pool_slots=4)
        m0 = trace.size()
        w.run_backward_sim(0, tf.SyntheticGradSource(5), 1)
        assert sum(e.bytes for e in trace.snapshot(m0) if e.kind == tf.EventKind.flush_end) == want
        w.close()


@pytest.mark.parametrize("hbm,h2d_split", [(0, 1), (1, 1), (2, 1), (1, 2), (2, 2)])
def test_hbm_retention_bits_and_pcie_bytes(tf, cuda, lock_dir, tmp_path, hbm, h2d_split):
    """Retained subgroups keep their state in HBM between phases: no D2H when
    retained, no H2D at the next update. Same bits and cache hits as the
    host-retention path and the oracle, including re-retention (C > M/2), a
    skipped iteration (same direction twice) and an op-level flush of an
    HBM-resident subgroup."""
    params = [100_000, 64_000, 99_996, 50_000, 77_777]
    seed, C = 23, 3
    trace = tf.EventTrace()
    tiers = [tf.Tier(tf.TierSpec(0, tf.TierKind.host_dram, "dram", 20e9, 20e9)),
             tf.Tier(tf.TierSpec(1, tf.TierKind.local_dir, str(tmp_path / "d"), 2e9, 2e9))]
    opt = (tf.ScheduleOptions(pool_slots=3, cache_slots=C, lock_dir=lock_dir) if hbm == 2 else
           tf.ScheduleOptions(pool_slots=C + 3, lock_dir=lock_dir))
    w = tf.OffloadWorker(0, tiers, opt, tf.AdamHyper(), trace, tf.DeviceOptions(0, 0, 0, 2, 0, 1, hbm, h2d_split))
    w.set_fixed_ratio([1.0, 1.0])
    for i, n in enumerate(params):
        w.add_subgroup(i, n)
    w.init_and_flush_all(seed)
    S = sum(params)
    applied = [0, 1, 2, 4]
    prev_retained = set()
    for it in applied:
        w.run_backward_sim(it, tf.SyntheticGradSource(seed))
        st = w.run_update(it)
        order = list(range(len(params))) if it % 2 == 0 else list(reversed(range(len(params))))
        retained = set(order[-C:])
        assert st.cache_hits == len(prev_retained)
        assert st.retained == C
        if hbm:
            assert st.h2d_bytes == 12 * (S - sum(params[i] for i in prev_retained))
            assert st.d2h_bytes == 12 * (S - sum(params[i] for i in retained))
        else:
            assert st.h2d_bytes == st.d2h_bytes == 12 * S
        prev_retained = retained
    want = {}
    for sg, n in enumerate(params):
        p, m, v = oracle.synthetic_params(n, seed, sg), np.zeros(n, np.float32), np.zeros(n, np.float32)
        for it in applied:
            p, m, v, p16, _ = oracle.adam_fused(p, m, v, oracle.synthetic_grads(n, seed, sg, it), 0, 0, it + 1)
        want[sg] = (np.concatenate([p, m, v]).view(np.uint32), p16)
    for sg in range(len(params)):
        assert np.array_equal(w.read_current_state(sg).view(np.uint32), want[sg][0]), sg
        assert np.array_equal(w.read_params16(sg), want[sg][1])
    # op-level flush of a retained (HBM-resident) subgroup writes the current bits
    w.enqueue_flush(3, 1).get()
    got = np.empty(3 * params[3], np.float32)
    tiers[1].read_subgroup(3, params[3], got)
    assert np.array_equal(got.view(np.uint32), want[3][0])
    assert np.array_equal(w.read_current_state(3).view(np.uint32), want[3][0])
    w.close()


def test_capacity_capped_tier_spills_and_keeps_bits(tf, cuda, lock_dir, tmp_path):
    """TierSpec.capacity_bytes ("host DRAM capped"): the host-DRAM
    tier holds at most its capacity in subgroups; Eq. 1 spills the rest to
    the other tiers by bandwidth; the state bits do not depend on placement."""
    params = [60_000] * 7 + [33_333]
    seed = 41
    block = 4096 * ((32 + 12 * 60_000 + 4095) // 4096)  # header + P||m||v of the largest, 4 KiB pages
    trace = tf.EventTrace()
    tiers = [tf.Tier(tf.TierSpec(0, tf.TierKind.host_dram, "dram", 50e9, 50e9, capacity_bytes=2 * block)),
             tf.Tier(tf.TierSpec(1, tf.TierKind.mem_throttled, "nvme", 400e6, 400e6)),
             tf.Tier(tf.TierSpec(2, tf.TierKind.local_dir, str(tmp_path / "remote"), 2e9, 2e9))]
    w = tf.OffloadWorker(0, tiers, tf.ScheduleOptions(pool_slots=4, lock_dir=lock_dir), tf.AdamHyper(), trace,
                         tf.DeviceOptions(0, 0, 0, 3))
    w.set_fixed_ratio([10.0, 2.0, 1.0])  # uncapped Eq. 1 would put most of the state on tier 0
    assert tf.assign_subgroups(7, [10.0, 2.0, 1.0]).counts[0] > 2
    for i, n in enumerate(params):
        w.add_subgroup(i, n)
    w.init_and_flush_all(seed)
    host, per_tier = w.residency_census()
    assert per_tier[0] <= 2 * 60_000 and sum(per_tier) == sum(params)
    for it in range(3):
        w.run_backward_sim(it, tf.SyntheticGradSource(seed))
        st = w.run_update(it)
        assert st.flush_allocation == tf.assign_subgroups_capped(len(params) - st.retained, [10.0, 2.0, 1.0],
                                                                 [2, -1, -1]).counts
        assert st.flush_allocation[0] <= 2
        host, per_tier = w.residency_census()
        assert per_tier[0] <= 2 * 60_000
    for sg, n in enumerate(params):
        p, m, v = oracle.synthetic_params(n, seed, sg), np.zeros(n, np.float32), np.zeros(n, np.float32)
        for it in range(3):
            p, m, v, p16, _ = oracle.adam_fused(p, m, v, oracle.synthetic_grads(n, seed, sg, it), 0, 0, it + 1)
        assert np.array_equal(w.read_current_state(sg).view(np.uint32), np.concatenate([p, m, v]).view(np.uint32))
        assert np.array_equal(w.read_params16(sg), p16)
    w.close()


@pytest.mark.parametrize("hbm", [2])
def test_full_size_subgroups_bit_exact(tf, cuda, lock_dir, tmp_path, hbm):
    """BASELINE shapes at full size: a 100M-param subgroup and the 7B shape's
    ragged last one (38,415,616), through host DRAM and an O_DIRECT directory
    tier with HBM retention, bit-exact against the oracle after 3 phases."""
    params = [100_000_000, 38_415_616]
    seed, iters = 42, 3
    trace = tf.EventTrace()
    tiers = [tf.Tier(tf.TierSpec(0, tf.TierKind.host_dram, "dram", 50e9, 50e9)),
             tf.Tier(tf.TierSpec(1, tf.TierKind.local_dir, str(tmp_path / "nvme"), 4e9, 4e9, io_parallelism=4))]
    opt = (tf.ScheduleOptions(pool_slots=3, cache_slots=1, lock_dir=lock_dir) if hbm == 2 else
           tf.ScheduleOptions(pool_slots=4, lock_dir=lock_dir))
    w = tf.OffloadWorker(0, tiers, opt, tf.AdamHyper(), trace, tf.DeviceOptions(0, 0, 0, 2, 0, 1, hbm))
    w.set_fixed_ratio([1.0, 1.0])
    for i, n in enumerate(params):
        w.add_subgroup(i, n)
    w.init_and_flush_all(seed)
    hits = []
    for it in range(iters):
        w.run_backward_sim(it, tf.SyntheticGradSource(seed))
        hits.append(w.run_update(it).cache_hits)
    assert hits == [0, 1, 1]
    for sg, n in enumerate(params):
        p, m, v = oracle.synthetic_params(n, seed, sg), np.zeros(n, np.float32), np.zeros(n, np.float32)
        for it in range(iters):
            p, m, v, p16, _ = oracle.adam_fused(p, m, v, oracle.synthetic_grads(n, seed, sg, it), 0, 0, it + 1)
        got = w.read_current_state(sg).view(np.uint32)
        assert np.array_equal(got[:n], p.view(np.uint32)), f"subgroup {sg} P"
        assert np.array_equal(got[n:2 * n], m.view(np.uint32)), f"subgroup {sg} m"
        assert np.array_equal(got[2 * n:], v.view(np.uint32)), f"subgroup {sg} v"
        assert np.array_equal(w.read_params16(sg), p16), f"subgroup {sg} params16"
        del p, m, v, p16, got
    w.close()


@pytest.mark.parametrize("hbm,skip", [(0, True), (1, True), (2, True), (0, False)])
def test_engine_returns_every_host_block(tf, cuda, lock_dir, tmp_path, hbm, skip):
    """Pool slots, host-DRAM blobs and spares, the write-back lane and the
    baseline flow's gradient stages are all freed once the engine and its
    tiers are gone."""
    import gc
    gc.collect()
    base = tf.host_blocks_live()
    tiers = [tf.Tier(tf.TierSpec(0, tf.TierKind.host_dram, "dram", 20e9, 20e9)),
             tf.Tier(tf.TierSpec(1, tf.TierKind.local_dir, str(tmp_path / "d"), 2e9, 2e9))]
    w = tf.OffloadWorker(0, tiers, tf.ScheduleOptions(pool_slots=4, cache_slots=2, lock_dir=lock_dir,
                                                      skip_gradients=skip),
                         tf.AdamHyper(), tf.EventTrace(), tf.DeviceOptions(0, 0, 0, 2, 0, 1, hbm))
    w.set_fixed_ratio([1.0, 1.0])
    for i in range(5):
        w.add_subgroup(i, 50_000 + 7 * i)
    w.init_and_flush_all(3)
    for it in range(3):
        w.run_backward_sim(it, tf.SyntheticGradSource(3))
        w.run_update(it)
    assert tf.host_blocks_live()[0] > base[0]
    w.close()
    del w, tiers
    gc.collect()
    assert tf.host_blocks_live() == base
    assert tf.host_block_free_failures() == 0


@pytest.mark.parametrize("hbm", [1, 2])
def test_tier_read_failure_surfaces_and_engine_stays_consistent(tf, cuda, lock_dir, tmp_path, hbm):
    """Fault injection (reference scheduler.hpp:689-693): a subgroup file that
    vanished from its directory tier fails its prefetch; run_update raises the
    tier's error, the subgroup stays on its tier, no slot is left mid-transfer,
    and the engine can be closed without leaking a host block."""
    import gc
    import os
    gc.collect()
    base = tf.host_blocks_live()
    params = [40_000] * 6
    tiers = [tf.Tier(tf.TierSpec(0, tf.TierKind.host_dram, "dram", 20e9, 20e9)),
             tf.Tier(tf.TierSpec(1, tf.TierKind.local_dir, str(tmp_path / "d"), 2e9, 2e9))]
    w = tf.OffloadWorker(0, tiers, tf.ScheduleOptions(pool_slots=4, cache_slots=1, lock_dir=lock_dir,
                                                      deadlock_timeout_s=10.0),
                         tf.AdamHyper(), tf.EventTrace(), tf.DeviceOptions(0, 0, 0, 2, 0, 1, hbm))
    w.set_fixed_ratio([1.0, 1.0])
    for i, n in enumerate(params):
        w.add_subgroup(i, n)
    w.init_and_flush_all(5)
    w.run_backward_sim(0, tf.SyntheticGradSource(5))
    w.run_update(0)
    on_dir = [sg for sg in range(len(params)) if w.meta(sg).residency == tf.Residency.on_tier and w.meta(sg).tier == 1]
    assert on_dir
    victim = on_dir[0]
    f = tmp_path / "d" / f"sg_{victim:06d}.bin"
    os.rename(f, str(f) + ".away")
    w.run_backward_sim(1, tf.SyntheticGradSource(5))
    with pytest.raises((tf.PlacementInconsistencyError, tf.IoError)):
        w.run_update(1)
    m = w.meta(victim)
    assert m.residency == tf.Residency.on_tier and m.tier == 1
    time.sleep(0.5)  # let the device work issued before the failure retire
    host, per_tier = w.residency_census()
    assert host + sum(per_tier) <= sum(params)
    assert all(w.pool_state(s)[0] != tf.SlotState.prefetching for s in range(4))
    w.close()
    del w, tiers
    gc.collect()
    assert tf.host_blocks_live() == base


def test_tier_write_failure_keeps_state_in_host_slots(tf, cuda, lock_dir, tmp_path):
    """Fault injection (reference scheduler.hpp:730-733): flushes to a tier
    whose directory vanished fail; run_update raises IoError and every
    subgroup that failed to flush is still host-cached in its slot with its
    updated state, so no state is lost."""
    import gc
    import shutil
    gc.collect()
    params = [30_000] * 5
    tiers = [tf.Tier(tf.TierSpec(0, tf.TierKind.host_dram, "dram", 20e9, 20e9)),
             tf.Tier(tf.TierSpec(1, tf.TierKind.local_dir, str(tmp_path / "d"), 2e9, 2e9))]
    w = tf.OffloadWorker(0, tiers, tf.ScheduleOptions(pool_slots=8, cache_slots=0, lock_dir=lock_dir,
                                                      deadlock_timeout_s=10.0),
                         tf.AdamHyper(), tf.EventTrace(), tf.DeviceOptions(0, 0, 0, 2, 0, 1, 0))
    w.set_fixed_ratio([1.0, 0.0])  # init: everything on host DRAM
    for i, n in enumerate(params):
        w.add_subgroup(i, n)
    w.init_and_flush_all(8)
    w.set_fixed_ratio([0.0, 1.0])  # phase 0 flushes everything to the directory tier ...
    shutil.rmtree(tmp_path / "d")  # ... which is gone
    (tmp_path / "d").write_text("not a directory")
    w.run_backward_sim(0, tf.SyntheticGradSource(8))
    with pytest.raises(tf.IoError):
        w.run_update(0)
    time.sleep(0.5)
    failed = [sg for sg in range(len(params)) if w.meta(sg).residency == tf.Residency.host_cached]
    assert failed  # their updated state stayed in the pool
    for sg in failed:
        n = params[sg]
        p, m, v, _, _ = oracle.adam_fused(oracle.synthetic_params(n, 8, sg), np.zeros(n, np.float32),
                                          np.zeros(n, np.float32), oracle.synthetic_grads(n, 8, sg, 0), 0, 0, 1)
        assert np.array_equal(w.read_current_state(sg).view(np.uint32), np.concatenate([p, m, v]).view(np.uint32))
    w.close()


def test_hbm_cache_writeback_failure_recovers(tf, cuda, lock_dir, tmp_path):
    """HBM cache mode: the write-back lane's flushes fail (tier directory
    gone); the written-back state survives in the lane's blocks or pool slots,
    reads back exactly, and once the tier is repaired the next phases run on
    and end bit-exact with the oracle (no subgroup lost or double-updated)."""
    import shutil
    params = [30_000, 31_000, 32_000, 33_000, 34_000, 35_000]
    seed = 12
    tiers = [tf.Tier(tf.TierSpec(0, tf.TierKind.host_dram, "dram", 20e9, 20e9)),
             tf.Tier(tf.TierSpec(1, tf.TierKind.local_dir, str(tmp_path / "d"), 2e9, 2e9))]
    w = tf.OffloadWorker(0, tiers, tf.ScheduleOptions(pool_slots=3, cache_slots=3, lock_dir=lock_dir,
                                                      deadlock_timeout_s=10.0),
                         tf.AdamHyper(), tf.EventTrace(), tf.DeviceOptions(0, 0, 0, 2, 0, 1, 2))
    w.set_fixed_ratio([1.0, 0.0])
    for i, n in enumerate(params):
        w.add_subgroup(i, n)
    w.init_and_flush_all(seed)

    def want(sg, steps):
        n = params[sg]
        p, m, v = oracle.synthetic_params(n, seed, sg), np.zeros(n, np.float32), np.zeros(n, np.float32)
        for it in range(steps):
            p, m, v, _, _ = oracle.adam_fused(p, m, v, oracle.synthetic_grads(n, seed, sg, it), 0, 0, it + 1)
        return np.concatenate([p, m, v]).view(np.uint32)

    w.run_backward_sim(0, tf.SyntheticGradSource(seed))
    w.run_update(0)  # ascending: 3, 4, 5 retained in HBM
    w.set_fixed_ratio([0.0, 1.0])
    shutil.rmtree(tmp_path / "d")
    (tmp_path / "d").write_text("not a directory")
    w.run_backward_sim(1, tf.SyntheticGradSource(seed))
    with pytest.raises(tf.IoError):
        w.run_update(1)  # descending: hits 5, 4, 3 written back through the lane -> fail
    time.sleep(0.5)
    for sg in (3, 4, 5):
        assert w.meta(sg).residency == tf.Residency.host_cached
        assert np.array_equal(w.read_current_state(sg).view(np.uint32), want(sg, 2))
    (tmp_path / "d").unlink()
    (tmp_path / "d").mkdir()
    w.set_fixed_ratio([1.0, 1.0])
    for it in (2, 3):
        w.run_backward_sim(it, tf.SyntheticGradSource(seed))
        w.run_update(it)
    for sg in range(len(params)):
        assert np.array_equal(w.read_current_state(sg).view(np.uint32), want(sg, 4)), sg
    w.close()


def test_two_level_cache_hbm_plus_host_slots(tf, cuda, lock_dir, tmp_path):
    """DeviceOptions.hbm_cache_slots < C: part of the retention capacity is
    held in HBM, the rest in host slots (two cache levels). Same hits and bits
    as the reference's host retention; fewer PCIe bytes than host-only
    retention, more than an all-HBM cache."""
    params = [50_000, 52_000, 54_000, 56_000, 58_000, 60_000]
    seed, C = 19, 4
    S = sum(params)

    def run(hbm, hbm_slots):
        tiers = [tf.Tier(tf.TierSpec(0, tf.TierKind.host_dram, "dram", 20e9, 20e9)),
                 tf.Tier(tf.TierSpec(1, tf.TierKind.local_dir, str(tmp_path / f"d{hbm}{hbm_slots}"), 2e9, 2e9))]
        w = tf.OffloadWorker(0, tiers, tf.ScheduleOptions(pool_slots=5, cache_slots=C, lock_dir=lock_dir),
                             tf.AdamHyper(), tf.EventTrace(),
                             tf.DeviceOptions(0, 0, 0, 2, 0, 1, hbm, 1, hbm_slots))
        w.set_fixed_ratio([1.0, 1.0])
        for i, n in enumerate(params):
            w.add_subgroup(i, n)
        w.init_and_flush_all(seed)
        hits, pcie = [], []
        for it in range(4):
            w.run_backward_sim(it, tf.SyntheticGradSource(seed))
            st = w.run_update(it)
            hits.append(st.cache_hits)
            pcie.append(st.h2d_bytes + st.d2h_bytes)
        states = [w.read_current_state(sg).view(np.uint32).copy() for sg in range(len(params))]
        w.close()
        return hits, pcie, states

    two_hits, two_pcie, two_states = run(2, 2)  # C = min(4, 2 + 5 - 3) = 4: 2 in HBM, 2 in host slots
    all_hits, all_pcie, _ = run(2, 0)
    host_hits, host_pcie, _ = run(0, 0)  # reference host retention: C = min(4, 5 - 3) = 2
    assert two_hits == all_hits == [0, C, C, C]
    assert host_hits == [0, 2, 2, 2]
    assert all(p < 2 * 12 * S for p in two_pcie[1:])
    assert all(a < t for a, t in zip(all_pcie[1:], two_pcie[1:]))
    for sg, n in enumerate(params):
        p, m, v = oracle.synthetic_params(n, seed, sg), np.zeros(n, np.float32), np.zeros(n, np.float32)
        for it in range(4):
            p, m, v, _, _ = oracle.adam_fused(p, m, v, oracle.synthetic_grads(n, seed, sg, it), 0, 0, it + 1)
        assert np.array_equal(two_states[sg], np.concatenate([p, m, v]).view(np.uint32)), sg


def test_reference_c1_shape_sampled(tf, cuda, lock_dir, tmp_path):
    """BASELINE configs[0] shape (1B params as 8 x 125M subgroups, host DRAM +
    one file tier, 3 Adam iterations, reference pool 5 / C = 2) through the
    engine. The inputs at 4096 sampled positions per subgroup come from the
    device generators (bit-exact with the oracle's, test_oracle_golden /
    test_kernel_parity), their Adam chain from the CPU oracle."""
    import torch
    n, M, seed, iters = 125_000_000, 8, 42, 3
    tiers = [tf.Tier(tf.TierSpec(0, tf.TierKind.host_dram, "dram", 20e9, 20e9)),
             tf.Tier(tf.TierSpec(1, tf.TierKind.local_dir, str(tmp_path / "d"), 2e9, 2e9, io_parallelism=4))]
    w = tf.OffloadWorker(0, tiers, tf.ScheduleOptions(pool_slots=5, lock_dir=lock_dir), tf.AdamHyper(),
                         tf.EventTrace(), tf.DeviceOptions(0, 0, 0, 3))
    w.set_fixed_ratio([1.0, 1.0])
    for sg in range(M):
        w.add_subgroup(sg, n)
    w.init_and_flush_all(seed)
    hits = []
    for it in range(iters):
        w.run_backward_sim(it, tf.SyntheticGradSource(seed))
        hits.append(w.run_update(it).cache_hits)
    assert hits == [0, 2, 2]  # reference survey probe of C1: hits 0/2/2
    idx = np.random.default_rng(3).integers(0, n, 4096)
    ti = torch.from_numpy(idx).to(cuda)
    p_d = torch.empty(n, device=cuda)
    z = torch.empty(n, device=cuda)
    g_d = torch.empty(n, dtype=torch.int16, device=cuda)
    for sg in range(M):
        tf.synthetic_state(p_d, z, z, seed, sg)
        p = p_d[ti].cpu().numpy()
        m = np.zeros(idx.size, np.float32)
        v = np.zeros(idx.size, np.float32)
        for it in range(iters):
            tf.synthetic_grads(g_d, seed, sg, it)
            g = g_d[ti].cpu().numpy().view(np.uint16)
            p, m, v, _, _ = oracle.adam_fused(p, m, v, g, 0, 0, it + 1)
        got = w.read_current_state(sg).view(np.uint32)
        assert np.array_equal(got[idx], p.view(np.uint32)), sg
        assert np.array_equal(got[n + idx], m.view(np.uint32)), sg
        assert np.array_equal(got[2 * n + idx], v.view(np.uint32)), sg
    w.close()


@pytest.mark.parametrize("kind,wd", [(0, 0.01), (1, 0.0), (1, 0.05)])
def test_everything_on_matches_oracle(tf, cuda, lock_dir, tmp_path, kind, wd):
    """All the B200 extensions at once: bf16 or f16 gradients and working
    params, AdamW, two-level HBM + host retention, a capacity-capped host-DRAM
    tier beside two directory tiers on one device semaphore, ragged subgroups,
    gradient accumulation, a skipped (non-finite) iteration. Bits and hits as
    the oracle says."""
    params = [70_001, 65_536, 33_333, 90_000, 12_345, 80_000, 44_444]
    seed, accum = 27, 2
    block = 4096 * ((32 + 12 * max(params) + 4095) // 4096)
    tiers = [tf.Tier(tf.TierSpec(0, tf.TierKind.host_dram, "dram", 50e9, 50e9, capacity_bytes=2 * block)),
             tf.Tier(tf.TierSpec(1, tf.TierKind.local_dir, str(tmp_path / "n"), 3e9, 3e9, io_parallelism=2,
                                 lock_device=1)),
             tf.Tier(tf.TierSpec(2, tf.TierKind.remote_dir, str(tmp_path / "r"), 1e9, 1e9, lock_device=1))]
    w = tf.OffloadWorker(0, tiers, tf.ScheduleOptions(pool_slots=5, cache_slots=4, lock_dir=lock_dir),
                         tf.AdamHyper(weight_decay=wd), tf.EventTrace(),
                         tf.DeviceOptions(0, kind, kind, 3, 0, 1, 2, 1, 2))
    w.set_fixed_ratio([5.0, 2.0, 1.0])
    for i, n in enumerate(params):
        w.add_subgroup(i, n)
    w.init_and_flush_all(seed)
    applied = []
    for it in range(5):
        w.run_backward_sim(it, tf.SyntheticGradSource(seed), accum)
        if it == 2:  # a poisoned gradient: the phase is rejected before any mutation
            import torch
            buf = torch.as_tensor(_DevView(w.grad_buffer(3), params[3]), device=cuda)
            buf[17] = 0x7C00 if kind == 0 else 0x7F80  # +Inf
            torch.cuda.synchronize()
            assert not w.gradients_finite()
            with pytest.raises(tf.GradientOverflowError):
                w.run_update(it)
            continue
        st = w.run_update(it)
        assert st.flush_allocation[0] <= 2
        applied.append(it)
    for sg, n in enumerate(params):
        p, m, v = oracle.synthetic_params(n, seed, sg), np.zeros(n, np.float32), np.zeros(n, np.float32)
        for it in applied:
            g = oracle.synthetic_grads(n, seed, sg, it, steps=accum, kind=kind)
            p, m, v, p16, _ = oracle.adam_fused(p, m, v, g, kind, kind, it + 1, weight_decay=wd)
        assert np.array_equal(w.read_current_state(sg).view(np.uint32), np.concatenate([p, m, v]).view(np.uint32)), sg
        assert np.array_equal(w.read_params16(sg), p16), sg
    w.close()


class _DevView:
    """__cuda_array_interface__ over an engine-owned 16-bit device buffer."""

    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<i2", "data": (ptr, False), "version": 3,
                                         "strides": None}


@pytest.mark.parametrize("hbm", [0, 2])
def test_tiny_ragged_subgroups_and_narrowing_overflow(tf, cuda, lock_dir, tmp_path, hbm):
    """Edge cases through the engine: subgroups of 1, 2, 3, 5 and 4099 params
    (scalar tails only / P % 4 != 0), and a learning rate large enough that
    the 16-bit working params overflow to Inf: PhaseStats.downscale_overflows
    equals the oracle's count and the bits still match."""
    params = [1, 2, 3, 5, 4099, 7]
    seed, lr = 33, 1.0e5
    tiers = [tf.Tier(tf.TierSpec(0, tf.TierKind.host_dram, "dram", 20e9, 20e9)),
             tf.Tier(tf.TierSpec(1, tf.TierKind.local_dir, str(tmp_path / "d"), 2e9, 2e9))]
    w = tf.OffloadWorker(0, tiers, tf.ScheduleOptions(pool_slots=4, cache_slots=2, lock_dir=lock_dir),
                         tf.AdamHyper(lr=lr), tf.EventTrace(), tf.DeviceOptions(0, 0, 0, 2, 0, 1, hbm))
    w.set_fixed_ratio([1.0, 1.0])
    for i, n in enumerate(params):
        w.add_subgroup(i, n)
    w.init_and_flush_all(seed)
    want = {sg: (oracle.synthetic_params(n, seed, sg), np.zeros(n, np.float32), np.zeros(n, np.float32))
            for sg, n in enumerate(params)}
    for it in range(3):
        w.run_backward_sim(it, tf.SyntheticGradSource(seed))
        st = w.run_update(it)
        over = 0
        for sg, n in enumerate(params):
            p, m, v = want[sg]
            p, m, v, p16, o = oracle.adam_fused(p, m, v, oracle.synthetic_grads(n, seed, sg, it), 0, 0, it + 1, lr=lr)
            want[sg] = (p, m, v)
            over += o
            if it == 2:
                assert np.array_equal(w.read_params16(sg), p16), sg
        assert st.downscale_overflows == over and over > 0
    for sg, n in enumerate(params):
        assert np.array_equal(w.read_current_state(sg).view(np.uint32), np.concatenate(want[sg]).view(np.uint32)), sg
    w.close()


@pytest.mark.parametrize("fixed", [True, False])
def test_cache_slots_lowered_to_zero_between_phases(tf, cuda, lock_dir, tmp_path, fixed):
    """set_cache_slots(0) after HBM-cache phases (the bench's streaming_c0),
    with the first C = 0 phase running in the same direction as the last
    retaining one (iteration 3 skipped), so its hits sit at the END of the
    order and are updated and flushed while the fetch frontier is still behind
    them: the frontier must not fetch them again (every later phase has no
    hits and nothing stays host-resident); bits stay the oracle's."""
    params = [60_000 + 8 * i for i in range(14)]
    seed, C = 19, 6
    tiers = [tf.Tier(tf.TierSpec(0, tf.TierKind.host_dram, "dram", 20e9, 20e9)),
             tf.Tier(tf.TierSpec(1, tf.TierKind.local_dir, str(tmp_path / "d"), 2e9, 2e9))]
    w = tf.OffloadWorker(0, tiers, tf.ScheduleOptions(pool_slots=5, cache_slots=C, lock_dir=lock_dir),
                         tf.AdamHyper(), tf.EventTrace(), tf.DeviceOptions(0, 0, 0, 3, 0, 1, 2))
    if fixed:
        w.set_fixed_ratio([3.0, 1.0])
    for i, n in enumerate(params):
        w.add_subgroup(i, n)
    w.init_and_flush_all(seed)
    hits = []
    applied = [0, 1, 2, 4, 5, 6, 7, 8]
    for it in applied:
        if it == 4:
            w.set_cache_slots(0)
        w.run_backward_sim(it, tf.SyntheticGradSource(seed))
        st = w.run_update(it)
        hits.append(st.cache_hits)
        host, _ = w.residency_census()
        if it >= 4:
            assert st.retained == 0 and host == 0, (it, st.retained, host)
    assert hits[:4] == [0, C, C, C] and hits[4:] == [0, 0, 0, 0], hits
    for sg, n in enumerate(params):
        p, m, v = oracle.synthetic_params(n, seed, sg), np.zeros(n, np.float32), np.zeros(n, np.float32)
        for it in applied:
            p, m, v, p16, _ = oracle.adam_fused(p, m, v, oracle.synthetic_grads(n, seed, sg, it), 0, 0, it + 1)
        assert np.array_equal(w.read_current_state(sg).view(np.uint32), np.concatenate([p, m, v]).view(np.uint32)), sg
    w.close()
