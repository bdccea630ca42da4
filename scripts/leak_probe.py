"""Host-block accounting through the smoke sequence, stage by stage (leak forensics)."""
import gc
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_02480_b200 import tierflow as tf  # noqa: E402

params = [200_003, 131_072, 77_777]
with tempfile.TemporaryDirectory() as tmp:
    trace = tf.EventTrace()
    tiers = [tf.Tier(tf.TierSpec(0, tf.TierKind.host_dram, "dram", 20e9, 20e9)),
             tf.Tier(tf.TierSpec(1, tf.TierKind.local_dir, os.path.join(tmp, "nvme"), 2e9, 2e9))]
    w = tf.OffloadWorker(0, tiers, tf.ScheduleOptions(pool_slots=4, lock_dir=os.path.join(tmp, "locks")),
                         tf.AdamHyper(), trace, tf.DeviceOptions(0))
    w.set_fixed_ratio([1.0, 1.0])
    for i, n in enumerate(params):
        w.add_subgroup(i, n)
    w.init_and_flush_all(5)
    print("after init", tf.host_blocks_live(), w.residency_census(), flush=True)
    for it in range(2):
        w.run_backward_sim(it, tf.SyntheticGradSource(5), 1)
        st = w.run_update(it)
        print("after phase", it, "hits", st.cache_hits, tf.host_blocks_live(), w.residency_census(), flush=True)
    w.close()
    print("after close", tf.host_blocks_live(), "tier refs", [sys.getrefcount(t) for t in tiers],
          "worker refs", sys.getrefcount(w), flush=True)
    for r in gc.get_referrers(w):
        desc = type(r).__name__
        if hasattr(r, "f_code"):
            desc += f" {r.f_code.co_name}:{r.f_lineno}"
        elif isinstance(r, dict):
            desc += " keys=" + ",".join(list(map(str, r.keys()))[:8])
        print("  referrer of w:", desc, flush=True)
    del w
    gc.collect()
    print("after del w", tf.host_blocks_live(), "tier refs", [sys.getrefcount(t) for t in tiers], flush=True)
    for t in tiers:
        t.close()
    print("after tier close", tf.host_blocks_live(), flush=True)
    print("referrers of dram tier:", [type(r).__name__ for r in gc.get_referrers(tiers[0])], flush=True)
    del tiers, trace
    gc.collect()
    print("after del tiers", tf.host_blocks_live(), flush=True)
