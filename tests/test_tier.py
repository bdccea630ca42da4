"""Storage tiers and tier locks through the C ABI (reference test_tier.cpp).
CPU only."""
import multiprocessing as mp
import os
import threading
import time

import numpy as np
import pytest


def _state(params, seed):
    return np.random.default_rng(seed).uniform(-5, 5, 3 * params).astype(np.float32)


@pytest.mark.parametrize("kind", ["local_dir", "mem_throttled", "host_dram"])
def test_round_trip_bitwise(tf, tmp_path, kind):
    k = tf.TierKind[kind]
    spec = tf.TierSpec(0, k, str(tmp_path / "t0"), 4e9, 4e9)
    t = tf.Tier(spec)
    P = 1000
    s = _state(P, 42)
    w = t.write_subgroup(5, P, s)
    assert w.bytes == 12 * P
    back = np.empty_like(s)
    r = t.read_subgroup(5, P, back)
    assert r.bytes == 12 * P
    assert np.array_equal(back.view(np.uint32), s.view(np.uint32))
    assert t.has_subgroup(5)
    t.remove_subgroup(5)
    assert not t.has_subgroup(5)


def test_file_format_v1(tf, tmp_path):
    # test_tier.cpp:51-95: 32-byte LE header "OPLM", v1, kind 0, id, count; file = 32 + 12P bytes
    t = tf.Tier(tf.TierSpec(0, tf.TierKind.local_dir, str(tmp_path)))
    P = 1000
    s = _state(P, 1)
    t.write_subgroup(77, P, s)
    f = tmp_path / "sg_000077.bin"
    raw = f.read_bytes()
    assert len(raw) == 32 + 12 * P
    assert raw[:4] == b"OPLM"
    assert int.from_bytes(raw[4:6], "little") == 1 and int.from_bytes(raw[6:8], "little") == 0
    assert int.from_bytes(raw[8:12], "little") == 77 and int.from_bytes(raw[12:20], "little") == P
    assert raw[20:32] == bytes(12)
    assert np.array_equal(np.frombuffer(raw[32:], np.float32), s)


def test_format_errors(tf, tmp_path):
    t = tf.Tier(tf.TierSpec(0, tf.TierKind.local_dir, str(tmp_path)))
    s = _state(100, 2)
    t.write_subgroup(3, 100, s)
    with pytest.raises(tf.FormatError):
        t.read_subgroup(3, 99, np.empty(297, np.float32))
    with pytest.raises(tf.PlacementInconsistencyError):
        t.read_subgroup(4, 100, np.empty(300, np.float32))
    p = tmp_path / "sg_000003.bin"
    raw = bytearray(p.read_bytes())
    raw[0] = 0
    p.write_bytes(bytes(raw))
    with pytest.raises(tf.FormatError):
        t.read_subgroup(3, 100, np.empty(300, np.float32))
    p.write_bytes(bytes(raw[:100]))
    with pytest.raises(tf.FormatError):
        t.read_subgroup(3, 100, np.empty(300, np.float32))


def test_mem_tier_grads_and_missing(tf):
    t = tf.Tier(tf.TierSpec(0, tf.TierKind.mem_throttled, "m", 4e9, 4e9))
    g = np.full(2000, 0.5, np.float32)
    t.write_grads(9, 2000, g)
    back = np.empty_like(g)
    t.read_grads(9, 2000, back)
    assert np.array_equal(back, g)
    with pytest.raises(tf.PlacementInconsistencyError):
        t.read_subgroup(1, 10, np.empty(30, np.float32))
    with pytest.raises(tf.ConfigError):
        tf.Tier(tf.TierSpec(0, tf.TierKind.mem_throttled, "m", 0.0, 1e9))


def test_throttle_rate_is_enforced(tf):
    # SPEC tier invariant: configured mem_throttled rates within +-10% on >= 4 MiB.
    t = tf.Tier(tf.TierSpec(0, tf.TierKind.mem_throttled, "m", 200e6, 100e6))
    P = 700_000  # 8.4 MB
    s = _state(P, 3)
    # The first write also allocates and page-faults the blob (host time, not
    # device time); measure the rewrite, as the reference's fidelity check is
    # otherwise flaky on slow hosts (proj/test_output.txt:15-25).
    t.write_subgroup(1, P, s)
    w = t.write_subgroup(1, P, s)
    r = t.read_subgroup(1, P, np.empty_like(s))
    assert 0.85 < (12 * P / w.seconds) / 100e6 < 1.1
    assert 0.85 < (12 * P / r.seconds) / 200e6 < 1.1
    pr = t.probe_bandwidth(8 << 20, 3)
    assert 0.85 < pr.read_bw / 200e6 < 1.15 and 0.85 < pr.write_bw / 100e6 < 1.15


def test_dir_probe_positive(tf, tmp_path):
    t = tf.Tier(tf.TierSpec(0, tf.TierKind.local_dir, str(tmp_path)))
    r = t.probe_bandwidth(4 << 20, 2)
    assert r.read_bw > 0 and r.write_bw > 0
    assert t.spec().read_bw == r.read_bw


def test_striped_dir_io(tf, tmp_path):
    t = tf.Tier(tf.TierSpec(0, tf.TierKind.remote_dir, str(tmp_path), io_parallelism=4))
    P = 1_000_003  # > 8 MiB payload: striped path, ragged size
    s = _state(P, 9)
    t.write_subgroup(2, P, s)
    back = np.empty_like(s)
    t.read_subgroup(2, P, back)
    assert np.array_equal(back.view(np.uint32), s.view(np.uint32))


def test_lock_guard_blocks_and_traces(tf, lock_dir):
    trace = tf.EventTrace()
    g = tf.acquire_tier_lock(lock_dir, 0, 99, trace)
    assert os.path.exists(tf.tier_lock_path(lock_dir, 0))
    got = []

    def contender():
        with tf.TierLockGuard(lock_dir, 0, 1, trace):
            got.append(time.monotonic_ns())

    th = threading.Thread(target=contender)
    th.start()
    time.sleep(0.1)
    released = time.monotonic_ns()
    g.release()
    th.join()
    assert got and got[0] >= released
    kinds = [e.kind for e in trace.snapshot()]
    assert kinds.count(tf.EventKind.lock_acquire) == 2 and kinds.count(tf.EventKind.lock_release) == 2


def _hold_lock(lock_dir, q, hold_s):
    from paper_2509_02480_b200 import tierflow as tf
    with tf.TierLockGuard(lock_dir, 1, 7):
        q.put(("in", time.monotonic_ns()))
        time.sleep(hold_s)
        q.put(("out", time.monotonic_ns()))


def test_lock_excludes_across_processes(tf, lock_dir):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_hold_lock, args=(lock_dir, q, 0.15)) for _ in range(3)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(30)
        assert p.exitcode == 0
    ev = sorted([q.get() for _ in range(6)], key=lambda x: x[1])
    depth = 0
    for kind, _ in ev:
        depth += 1 if kind == "in" else -1
        assert depth <= 1


def test_semaphore_width_admits_two(tf, lock_dir):
    a = tf.TierLockGuard(lock_dir, 2, 0, width=2)
    done = threading.Event()

    def second():
        with tf.TierLockGuard(lock_dir, 2, 1, width=2):
            done.set()

    th = threading.Thread(target=second)
    th.start()
    assert done.wait(5.0)
    th.join()
    a.release()


def test_host_dram_tier_blocks_are_freed(tf):
    """Host-block accounting: a host-DRAM tier's blobs and spares are returned
    when the tier goes away (no pinned memory leaks across engines)."""
    import gc
    gc.collect()
    base = tf.host_blocks_live()
    t = tf.Tier(tf.TierSpec(0, tf.TierKind.host_dram, "dram", 1e9, 1e9))
    P = 10_000
    for sg in range(5):
        t.write_subgroup(sg, P, _state(P, sg))
    back = np.empty(3 * P, np.float32)
    t.read_subgroup(3, P, back)
    t.remove_subgroup(2)
    assert tf.host_blocks_live()[0] > base[0]
    del t
    gc.collect()
    assert tf.host_blocks_live() == base
