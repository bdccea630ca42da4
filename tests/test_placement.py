"""Product placement/ordering functions (C ABI, host) against the oracle and
the reference known answers. CPU only."""
import numpy as np
import pytest

import oracle


def test_assign_subgroups_matches_oracle_and_golden(tf, golden):
    for M, bw, counts in zip(golden["eq1_M"], golden["eq1_bw"], golden["eq1_counts"]):
        n = int((bw >= 0).sum())
        got = tf.assign_subgroups(int(M), bw[:n].tolist()).counts
        assert got == counts[:n].tolist()
    rng = np.random.default_rng(3)
    for _ in range(500):
        N = int(rng.integers(1, 5))
        M = int(rng.integers(1, 200))
        bw = [float(x) for x in np.where(rng.random(N) < 0.1, 0.0, 10 ** rng.uniform(-2, 2, N))]
        if not any(bw):
            bw[0] = 1.0
        assert tf.assign_subgroups(M, bw).counts == oracle.assign_subgroups(M, bw)


def test_assign_subgroups_properties(tf):
    # test_placement.cpp:81-103: scale invariance and monotonicity.
    rng = np.random.default_rng(5)
    for _ in range(100):
        M = int(rng.integers(1, 41))
        B = rng.uniform(0.1, 50.0, 3).tolist()
        a = tf.assign_subgroups(M, B).counts
        for c in (0.5, 2.0, 1024.0, 3.7):
            assert tf.assign_subgroups(M, [b * c for b in B]).counts == a
        boosted = list(B)
        boosted[1] *= 1.7
        assert tf.assign_subgroups(M, boosted).counts[1] >= a[1]
    assert tf.assign_subgroups(12, [2.0, 1.0]).counts == [8, 4]


def test_destination_plan_matches_oracle(tf):
    rng = np.random.default_rng(11)
    for _ in range(300):
        N = int(rng.integers(1, 5))
        M = int(rng.integers(1, 40))
        bw = [float(x) for x in 10 ** rng.uniform(-1, 1, N)]
        cap = int(rng.integers(0, M + 3))
        order = rng.permutation(M).tolist()
        plan = tf.DestinationPlan(order, cap, bw)
        r, t, a = oracle.destination_plan(M, cap, bw)
        for k, sg in enumerate(order):
            got = plan.assign_storage_tier(sg)
            assert (int(got.host_retain), got.tier) == (r[k], t[k])
        assert plan.flush_allocation().counts == a
        assert plan.retained_count() == sum(r)


def test_update_plan_alternates(tf):
    # test_scheduler.cpp:127-142
    even = tf.UpdatePlan.make(0, [0, 1, 2, 3], True)
    odd = tf.UpdatePlan.make(1, [0, 1, 2, 3], True)
    assert even.order == [0, 1, 2, 3] and even.ascending
    assert odd.order == [3, 2, 1, 0] and not odd.ascending
    assert tf.UpdatePlan.make(1, [0, 1, 2, 3], False).ascending
    assert even.next_after(2) == 3 and even.next_after(3) is None
    assert odd.next_after(3) == 2 and odd.next_after(0) is None


def test_retention_capacity(tf):
    for caching in (0, 1):
        for pool in range(3, 12):
            for cache in range(-1, 10):
                for M in range(0, 12):
                    assert tf.retention_capacity(bool(caching), pool, cache, M) == \
                        oracle.lib().orc_retention_capacity(caching, pool, cache, M)


def test_ema_arithmetic(tf):
    # test_placement.cpp:122-167
    est = tf.BandwidthEstimate([200e6], [200e6], 1.0)
    tf.update_bandwidth_estimates(est, [tf.TierObservation(2, 300e6, 2.0, 2, 300e6, 2.0)])
    assert abs(est.effective(0) - 150e6) < 1 and est.sample_count[0] == 4
    est = tf.BandwidthEstimate([200e6, 64e6], [100e6, 64e6], 0.5)
    tf.update_bandwidth_estimates(est, [tf.TierObservation(1, 50e6, 1.0, 0, 0, 0), tf.TierObservation()])
    assert abs(est.read_bw[0] - 125e6) < 1 and est.write_bw[0] == 100e6 and est.effective(1) == 64e6


def test_rebalance_after_bandwidth_drop(tf):
    # test_placement.cpp:187-211 (acceptance criterion 11)
    est = tf.BandwidthEstimate([200e6, 200e6], [200e6, 200e6], 0.5)
    before = tf.assign_subgroups(16, est.effective_all()).counts[1]
    obs = [tf.TierObservation(1, 200e6, 1.0, 1, 200e6, 1.0), tf.TierObservation(1, 100e6, 1.0, 1, 100e6, 1.0)]
    tf.update_bandwidth_estimates(est, obs)
    after1 = tf.assign_subgroups(16, est.effective_all()).counts[1]
    tf.update_bandwidth_estimates(est, obs)
    after2 = tf.assign_subgroups(16, est.effective_all()).counts[1]
    assert after1 <= before and after2 < before


def _paper_scale_cases():
    """SURVEY §8 shapes: C2 68 subgroups, C3 200 over 1/2/4/8 ranks, C4 690
    over 1/8 ranks (86/87 per rank), C5 sweep extremes; two- and three-tier
    bandwidth vectors from the paper's testbeds (GB/s:
    host DRAM ~25-55, NVMe 5.3-6.9, PFS 3.6-13.7)."""
    from paper_2509_02480_b200 import parallel
    Ms = {68, 200, 690, 9, 78}  # 9 = 1B at 125M per subgroup; 78 = 5B at 64M
    for M, worlds in ((200, (2, 4, 8)), (690, (8,)), (68, (8,))):
        for w in worlds:
            Ms.update(parallel.shard(M, w, r)[1] for r in range(w))
    bws = [[55.0, 5.3], [25.0, 6.9], [55.0, 5.3, 3.6], [6.9, 3.6], [5.3, 13.7], [25.0, 6.9, 4.8], [1.0, 1.0, 1.0]]
    for M in sorted(Ms):
        for bw in bws:
            yield M, bw


def test_paper_scale_placement_matches_oracle_and_reference(tf):
    R = oracle.ref() if oracle.ref_available() else None
    rng = np.random.default_rng(17)
    for M, bw in _paper_scale_cases():
        want = oracle.assign_subgroups(M, bw)
        assert tf.assign_subgroups(M, bw).counts == want, (M, bw)
        assert sum(want) == M
        if R is not None:
            counts = np.zeros(len(bw), np.int32)
            assert R.ref_assign_subgroups(M, np.asarray(bw, np.float64), len(bw), counts) == 0
            assert counts.tolist() == want, (M, bw)
        for cap in (0, 5, 13, 29, M // 2):
            order = list(range(M)) if rng.random() < 0.5 else list(reversed(range(M)))
            plan = tf.DestinationPlan(order, cap, bw)
            r, t, a = oracle.destination_plan(M, cap, bw)
            got = [plan.assign_storage_tier(sg) for sg in order]
            assert [(int(g.host_retain), g.tier) for g in got] == list(zip(r, t)), (M, bw, cap)
            assert plan.flush_allocation().counts == a
            if R is not None:
                rr, tt, aa = (np.zeros(M, np.int32), np.zeros(M, np.int32), np.zeros(len(bw), np.int32))
                assert R.ref_destination_plan(np.asarray(order, np.uint32), M, cap, np.asarray(bw, np.float64),
                                              len(bw), rr, tt, aa) == 0
                assert rr.tolist() == r and tt.tolist() == t and aa.tolist() == a


def _brute_capped(M, bw, caps):
    """min over T (sum M, T_i <= caps_i, T_i = 0 where B_i = 0) of max T_i/B_i."""
    import itertools
    N = len(bw)
    best = None
    ranges = [range(0, (min(M, c) if c >= 0 else M) + 1) if b > 0 else range(1) for b, c in zip(bw, caps)]
    for T in itertools.product(*ranges):
        if sum(T) != M:
            continue
        v = max(T[i] / bw[i] for i in range(N) if bw[i] > 0)
        best = v if best is None else min(best, v)
    return best


def test_capped_eq1_equals_reference_when_caps_do_not_bind(tf):
    rng = np.random.default_rng(23)
    for _ in range(300):
        N = int(rng.integers(1, 4))
        M = int(rng.integers(1, 120))
        bw = [float(x) for x in 10 ** rng.uniform(-1, 1, N)]
        ref = oracle.assign_subgroups(M, bw)
        caps = [c + int(rng.integers(0, 5)) if rng.random() < 0.7 else -1 for c in ref]
        assert tf.assign_subgroups_capped(M, bw, caps).counts == ref


def test_capped_eq1_respects_caps_and_is_minmax_optimal(tf):
    rng = np.random.default_rng(29)
    checked = 0
    for _ in range(400):
        N = int(rng.integers(2, 4))
        M = int(rng.integers(1, 25))
        bw = [float(x) for x in 10 ** rng.uniform(-1, 1, N)]
        caps = [int(rng.integers(0, M + 1)) if rng.random() < 0.6 else -1 for _ in range(N)]
        room = sum(M if c < 0 else c for c in caps)
        if room < M:
            with pytest.raises(tf.ConfigError):
                tf.assign_subgroups_capped(M, bw, caps)
            continue
        got = tf.assign_subgroups_capped(M, bw, caps).counts
        assert sum(got) == M
        assert all(c < 0 or g <= c for g, c in zip(got, caps))
        opt = _brute_capped(M, bw, caps)
        assert max(g / b for g, b in zip(got, bw) if b > 0) == pytest.approx(opt, rel=1e-12)
        checked += 1
    assert checked > 100
    # C4-style: a fast host-DRAM tier capped, the rest spills to NVMe and remote by bandwidth
    assert tf.assign_subgroups_capped(690, [50.0, 6.9, 3.6], [100, -1, -1]).counts == [100, 388, 202]
