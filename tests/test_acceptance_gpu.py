"""The reference acceptance criteria that exercise the update phase
(reference tests/acceptance.cpp), run against the B200 engine on throttled
in-memory tiers whose ground truth is the configured rate (-m gpu)."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def run_bench(tf, tier_rates, sub_params, n_sub, iterations, *, lock_dir, pool_slots=4, cache_slots=-1,
              multi_path=True, workers=1, warmup=0, before_iteration=None, seed=424242):
    """A thread-per-worker harness in the shape of BenchRunner::run
    (harness.hpp:45-67, 194-255): backward sim -> finite check -> update."""
    trace = tf.EventTrace()
    tiers = [tf.Tier(tf.TierSpec(i, tf.TierKind.mem_throttled, f"mem{i}", r * 1e6, w * 1e6))
             for i, (r, w) in enumerate(tier_rates)]
    opt = tf.ScheduleOptions(pool_slots=pool_slots, cache_slots=cache_slots, multi_path=multi_path, lock_dir=lock_dir)
    engines = []
    for w in range(workers):
        e = tf.OffloadWorker(w, tiers, opt, tf.AdamHyper(), trace, tf.DeviceOptions(0))
        base, rem = divmod(n_sub, workers)
        begin = w * base + min(w, rem)
        for k in range(base + (w < rem)):
            e.add_subgroup(begin + k, sub_params)
        e.init_and_flush_all(seed)
        engines.append(e)
    src = tf.SyntheticGradSource(seed)
    iters = []
    for it in range(iterations):
        if before_iteration:
            before_iteration(it, tiers)
        for e in engines:
            e.run_backward_sim(it, src, 1)
        stats = [None] * workers
        import time
        t0 = time.perf_counter()
        ths = [threading.Thread(target=lambda i=i: stats.__setitem__(i, engines[i].run_update(it)))
               for i in range(workers)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        update_s = time.perf_counter() - t0
        alloc = np.sum([s.flush_allocation for s in stats], axis=0).tolist()
        iters.append(dict(update_s=update_s, alloc=alloc, hits=sum(s.cache_hits for s in stats), stats=stats,
                          warmup=it < warmup))
    for e in engines:
        e.close()
    return iters, trace


def mean_update(iters):
    xs = [r["update_s"] for r in iters if not r["warmup"]]
    return sum(xs) / len(xs)


def test_c8_multipath_speedup(tf, cuda, lock_dir):
    # acceptance.cpp:377-410: 200+100 MB/s tiers vs tier 0 alone, C = 0, ratio <= 0.77 (ideal 0.667)
    kw = dict(pool_slots=4, cache_slots=0, warmup=1, lock_dir=lock_dir)
    multi, _ = run_bench(tf, [(200, 200), (100, 100)], 350_000, 12, 4, multi_path=True, **kw)
    single, _ = run_bench(tf, [(200, 200), (100, 100)], 350_000, 12, 4, multi_path=False, **kw)
    ratio = mean_update(multi) / mean_update(single)
    assert ratio <= 0.77, ratio


def test_c9_tier_completion_balance(tf, cuda, lock_dir):
    # acceptance.cpp:415-440: per-tier busy time spread <= 25% under Eq. 1
    _, trace = run_bench(tf, [(200, 200), (100, 100)], 350_000, 12, 4, pool_slots=4, cache_slots=0,
                         lock_dir=lock_dir)
    busy, opened = {0: 0.0, 1: 0.0}, {}
    for e in trace.snapshot():
        if e.kind in (tf.EventKind.prefetch_start, tf.EventKind.flush_start):
            opened[(e.subgroup_id, e.tier_id)] = e.timestamp_ns
        elif e.kind in (tf.EventKind.prefetch_end, tf.EventKind.flush_end):
            busy[e.tier_id] += (e.timestamp_ns - opened[(e.subgroup_id, e.tier_id)]) / 1e9
    hi, lo = max(busy.values()), min(busy.values())
    assert (hi - lo) / hi <= 0.25, busy


def test_c11_adaptive_rebalance(tf, cuda, lock_dir):
    # acceptance.cpp:500-530: tier 1 drops 200 -> 50 MB/s before iteration 3;
    # its flush allocation strictly decreases within two iterations and does not bounce back.
    def drop(it, tiers):
        if it == 3:
            tiers[1].set_throttle_rates(50e6, 50e6)
    iters, _ = run_bench(tf, [(200, 200), (200, 200)], 250_000, 16, 6, pool_slots=4, cache_slots=0,
                         lock_dir=lock_dir, before_iteration=drop)
    a = [r["alloc"][1] for r in iters]
    assert a[4] < a[2] or a[5] < a[2], a
    assert a[5] <= a[4], a


def test_c12_effective_io_definition(tf, cuda, lock_dir):
    # acceptance.cpp:535-580: per-subgroup 2*size/(t_r + t_w) from the raw trace equals PhaseStats.subgroup_io
    iters, trace = run_bench(tf, [(300, 300), (150, 150)], 100_000, 8, 1, pool_slots=6, cache_slots=0,
                             lock_dir=lock_dir)
    st = iters[0]["stats"][0]
    opened, per = {}, {}
    for e in trace.snapshot():
        key = (e.subgroup_id, int(e.kind))
        if e.kind in (tf.EventKind.prefetch_start, tf.EventKind.flush_start):
            opened[key] = e.timestamp_ns
        elif e.kind == tf.EventKind.prefetch_end:
            per.setdefault(e.subgroup_id, [0.0, 0.0])[0] += (e.timestamp_ns - opened[(e.subgroup_id, 0)]) / 1e9
        elif e.kind == tf.EventKind.flush_end:
            per.setdefault(e.subgroup_id, [0.0, 0.0])[1] += (e.timestamp_ns - opened[(e.subgroup_id, 4)]) / 1e9
    size = 12.0 * 100_000
    hand = np.mean([2 * size / (r + w) for r, w in per.values()])
    metric = np.mean([2 * s.state_bytes / (s.read_seconds + s.write_seconds) for s in st.subgroup_io
                      if s.fetched and s.flushed])
    assert len(per) == 8 and abs(metric - hand) / hand < 1e-9


def test_c7_lock_exclusivity_four_workers(tf, cuda, lock_dir):
    # acceptance.cpp:306-372 (thread mode): 4 workers x 2 tiers, >= 200 lock ops, no overlap per tier
    _, trace = run_bench(tf, [(1000, 1000), (600, 600)], 20_000, 24, 5, pool_slots=3, workers=4,
                         lock_dir=lock_dir)
    per, opened, n = {}, {}, 0
    for e in trace.snapshot():
        if e.kind == tf.EventKind.lock_acquire:
            opened[(e.tier_id, e.worker_id)] = e.timestamp_ns
            n += 1
        elif e.kind == tf.EventKind.lock_release:
            per.setdefault(e.tier_id, []).append((opened.pop((e.tier_id, e.worker_id)), e.timestamp_ns))
    assert n >= 200
    for iv in per.values():
        iv.sort()
        assert all(iv[i][1] <= iv[i + 1][0] for i in range(len(iv) - 1))


def test_c5_cache_hits_engine_harness(tf, cuda, lock_dir):
    # acceptance.cpp:246-272 through the harness shape: hits 0,4,4,4 with C = 4, M = 12
    iters, trace = run_bench(tf, [(300, 300), (150, 150)], 20_000, 12, 4, pool_slots=7, lock_dir=lock_dir)
    assert [r["hits"] for r in iters] == [0, 4, 4, 4]
    assert sum(1 for e in trace.snapshot() if e.kind == tf.EventKind.cache_hit) == 12


def test_c10_ablation_monotonicity(tf, cuda, lock_dir):
    # acceptance.cpp:445-490: the four §4.6 flags enabled progressively; mean
    # update time non-increasing within a 5% band, all-on the fastest.
    def ladder(step):
        trace = tf.EventTrace()
        tiers = [tf.Tier(tf.TierSpec(0, tf.TierKind.mem_throttled, "m0", 200e6, 200e6)),
                 tf.Tier(tf.TierSpec(1, tf.TierKind.mem_throttled, "m1", 100e6, 100e6))]
        opt = tf.ScheduleOptions(pool_slots=5, lock_dir=lock_dir, enable_caching=step >= 1, skip_gradients=step >= 2,
                                 atomic_rw=step >= 3, multi_path=step >= 4)
        engines = []
        for w in range(2):
            e = tf.OffloadWorker(w, tiers, opt, tf.AdamHyper(), trace, tf.DeviceOptions(0))
            for k in range(8):
                e.add_subgroup(w * 8 + k, 1_000_000)
            e.init_and_flush_all(424242)
            engines.append(e)
        import time
        times = []
        for it in range(4):
            for e in engines:
                e.run_backward_sim(it, tf.SyntheticGradSource(424242), 1)
            t0 = time.perf_counter()
            ths = [threading.Thread(target=e.run_update, args=(it,)) for e in engines]
            for t in ths:
                t.start()
            for t in ths:
                t.join()
            times.append(time.perf_counter() - t0)
        for e in engines:
            e.close()
        return sum(times[1:]) / 3
    t = [ladder(s) for s in range(5)]
    for i in range(4):
        assert t[i + 1] <= t[i] * 1.05, t
    assert t[4] <= min(t) * 1.0 + 1e-12, t
