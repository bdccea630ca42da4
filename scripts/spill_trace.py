"""Spill-configuration phase traces: the engine's event trace of one update
phase on two directory tiers (capped pool, HBM cache), reduced to per-tier
I/O intervals, disk busy time (union over tiers) and idle gaps.

    python scripts/spill_trace.py [subgroups=12] [pool=8] [cache=6] [io_par=4] [hbm=2]
"""
import json
import os
import shutil
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2509_02480_b200 import tierflow as tf  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 12
pool = int(sys.argv[2]) if len(sys.argv) > 2 else 8
cache = int(sys.argv[3]) if len(sys.argv) > 3 else 6
iopar = int(sys.argv[4]) if len(sys.argv) > 4 else 4
hbm = int(sys.argv[5]) if len(sys.argv) > 5 else 2
lock_device = int(sys.argv[6]) if len(sys.argv) > 6 else 0
dram_cap = int(sys.argv[7]) if len(sys.argv) > 7 else 0  # > 0: a host-DRAM tier capped at this many subgroups
hbm_slots = int(sys.argv[8]) if len(sys.argv) > 8 else 0  # > 0: two-level cache, this many of C in HBM
root = ROOT / "gpurun_out" / "spill_trace_tiers"
shutil.rmtree(root, ignore_errors=True)
off = 1 if dram_cap > 0 else 0
tiers = [tf.Tier(tf.TierSpec(off, tf.TierKind.local_dir, str(root / "nvme"), 0, 0, io_parallelism=iopar,
                             lock_device=lock_device)),
         tf.Tier(tf.TierSpec(off + 1, tf.TierKind.remote_dir, str(root / "remote"), 0, 0, io_parallelism=iopar,
                             lock_device=lock_device))]
if dram_cap > 0:
    block = 4096 * ((32 + 12 * 100_000_000 + 4095) // 4096)
    tiers = [tf.Tier(tf.TierSpec(0, tf.TierKind.host_dram, "dram", 50e9, 50e9, capacity_bytes=dram_cap * block))] + tiers
for t in tiers:
    if t.spec().kind == tf.TierKind.host_dram:
        continue
    pr = t.probe_bandwidth(1 << 30, 3)
    print(f"tier {t.id()} probe r={pr.read_bw / 1e9:.2f} w={pr.write_bw / 1e9:.2f}", flush=True)
trace = tf.EventTrace()
w = tf.OffloadWorker(0, tiers, tf.ScheduleOptions(pool_slots=pool, cache_slots=cache, lock_dir=str(root / "locks")),
                     tf.AdamHyper(), trace, tf.DeviceOptions(0, 0, 0, 4, 0, 1, hbm, 1, hbm_slots))
for k in range(M):
    w.add_subgroup(k, 100_000_000)
w.init_and_flush_all(42)
out = []
for it in range(5):
    w.run_backward_sim(it, tf.SyntheticGradSource(42))
    torch.cuda.synchronize()
    mark = trace.size()
    st = w.run_update(it)
    ev = trace.snapshot(mark)
    t0 = ev[0].timestamp_ns
    open_ = {}
    iv = []
    locks = []
    for e in ev:
        key = (e.subgroup_id, e.tier_id)
        if e.kind in (tf.EventKind.prefetch_start, tf.EventKind.flush_start):
            open_[(key, e.kind)] = e.timestamp_ns
        elif e.kind == tf.EventKind.lock_acquire:
            open_[(("L", e.tier_id, e.worker_id), e.kind)] = e.timestamp_ns
        elif e.kind == tf.EventKind.lock_release:
            s = open_.pop((("L", e.tier_id, e.worker_id), tf.EventKind.lock_acquire), None)
            if s is not None:
                locks.append(("L", -1, e.tier_id, (s - t0) / 1e6, (e.timestamp_ns - t0) / 1e6))
        elif e.kind in (tf.EventKind.prefetch_end, tf.EventKind.flush_end):
            k0 = tf.EventKind.prefetch_start if e.kind == tf.EventKind.prefetch_end else tf.EventKind.flush_start
            s = open_.pop((key, k0), None)
            if s is not None:
                iv.append(("R" if e.kind == tf.EventKind.prefetch_end else "W", e.subgroup_id, e.tier_id,
                           (s - t0) / 1e6, (e.timestamp_ns - t0) / 1e6))
    iv.sort(key=lambda x: x[3])
    span = (ev[-1].timestamp_ns - t0) / 1e6
    # union of I/O intervals over both tiers = time the disk had work
    busy, cur = 0.0, None
    for _, _, _, a, b in iv:
        if cur is None or a > cur[1]:
            if cur:
                busy += cur[1] - cur[0]
            cur = [a, b]
        else:
            cur[1] = max(cur[1], b)
    if cur:
        busy += cur[1] - cur[0]
    print(f"phase {it}: {st.wall_seconds * 1e3:.0f} ms, io busy(union) {busy:.0f} ms, hits {st.cache_hits}", flush=True)
    for x in sorted(iv + locks, key=lambda x: x[3]):
        print(f"   {x[0]} sg{x[1]:3d} tier{x[2]} {x[3]:8.0f} -> {x[4]:8.0f} ({x[4] - x[3]:6.0f} ms)")
    out.append(dict(phase=it, wall_ms=st.wall_seconds * 1e3, busy_ms=busy, intervals=iv))
w.close()
shutil.rmtree(root, ignore_errors=True)
Path("gpurun_out/spill_trace.json").write_text(json.dumps(out, indent=1))
