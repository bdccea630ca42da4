"""End-to-end update-phase pipeline sweep on the Llama-2-7B-shaped state:
host_dram + local_dir tiers, varying pool slots / retention / ring depth.
Prints per-phase time, PCIe-stream busy fractions and pipeline gaps from the
engine's per-subgroup timeline, and writes gpurun_out/e2e_sweep.json.

    python scripts/e2e_sweep.py [total_params] [configs...]
        config = pool:cache:ring:zero_copy:d2h_split[:hbm_retain[:h2d_split]]
"""
import json
import shutil
import statistics
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2509_02480_b200 import tierflow as tf  # noqa: E402

total = int(sys.argv[1]) if len(sys.argv) > 1 else 6_738_415_616
configs = [tuple(int(x) for x in c.split(":")) for c in sys.argv[2:]] or [(12, 5, 3, 0, 1, 1), (12, 5, 3, 0, 1, 0)]
configs = [c if len(c) >= 6 else c + (1,) for c in configs]
configs = [c if len(c) == 7 else c + (1,) for c in configs]
sub = 100_000_000
sizes = [min(sub, total - k * sub) for k in range((total + sub - 1) // sub)]
import os
root = ROOT / "gpurun_out" / "e2e_sweep_tiers"
shutil.rmtree(root, ignore_errors=True)
# TFB_TIERS: "dram,nvme" (default) or "nvme,remote" (host DRAM only as pool
# slots: the state spills to the directory tiers)
tier_set = os.environ.get("TFB_TIERS", "dram,nvme").split(",")
remote_root = Path(os.environ.get("TFB_REMOTE_ROOT", "/tmp/tfb_remote"))
shutil.rmtree(remote_root, ignore_errors=True)
tiers = []
for name in tier_set:
    tid = len(tiers)
    if name == "dram":
        tiers.append(tf.Tier(tf.TierSpec(tid, tf.TierKind.host_dram, "dram", 50e9, 50e9)))
    elif name == "nvme":
        tiers.append(tf.Tier(tf.TierSpec(tid, tf.TierKind.local_dir, str(root / "nvme"), 0, 0, io_parallelism=4)))
    elif name == "remote":
        tiers.append(tf.Tier(tf.TierSpec(tid, tf.TierKind.remote_dir, str(remote_root), 0, 0, io_parallelism=4)))
    else:
        raise SystemExit(f"unknown tier {name}")
    if name != "dram":
        pr = tiers[-1].probe_bandwidth(1 << 30, 3)
        print(f"{name} probe r={pr.read_bw/1e9:.2f} w={pr.write_bw/1e9:.2f} GB/s", flush=True)
out = []
for pool, cache, ring, zc, split, hbm, hsplit in configs:
    trace = tf.EventTrace()
    w = tf.OffloadWorker(0, tiers, tf.ScheduleOptions(pool_slots=pool, cache_slots=cache,
                                                            lock_dir=str(root / "locks")),
                         tf.AdamHyper(), trace, tf.DeviceOptions(0, 0, 0, ring, zc, split, hbm, hsplit))
    for k, n in enumerate(sizes):
        w.add_subgroup(k, n)
    t0 = time.time()
    w.init_and_flush_all(42)
    init_s = time.time() - t0
    phases = []
    for it in range(7):
        w.run_backward_sim(it, tf.SyntheticGradSource(42))
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        st = w.run_update(it)
        ms = (time.perf_counter() - t1) * 1e3
        tl = w.last_timeline()
        h2d_busy = sum(s["h2d_end"] - s["h2d_start"] for s in tl)
        d2h_busy = sum(s["d2h_end"] - max(s["k_end"], (tl[i - 1]["d2h_end"] if i else 0)) for i, s in enumerate(tl))
        h2d_gaps = sum(max(0.0, tl[i + 1]["h2d_start"] - tl[i]["h2d_end"]) for i in range(len(tl) - 1))
        span = tl[-1]["d2h_end"]
        phases.append(dict(ms=ms, span=span, h2d_busy=h2d_busy, d2h_busy=d2h_busy, h2d_gaps=h2d_gaps,
                           hits=st.cache_hits, alloc=st.flush_allocation, kernel_ms=st.kernel_seconds * 1e3,
                           h2d_bytes=st.h2d_bytes, d2h_bytes=st.d2h_bytes))
        print(f"pool={pool} cache={cache} ring={ring} zc={zc} split={split} hbm={hbm} h2dsplit={hsplit} phase {it}: {ms:7.1f} ms (device span {span:7.1f}) "
              f"h2d busy {h2d_busy:7.1f} gaps {h2d_gaps:6.1f} d2h busy {d2h_busy:7.1f} hits {st.cache_hits} "
              f"alloc {st.flush_allocation} h2d {st.h2d_bytes/1e9:.1f} GB d2h {st.d2h_bytes/1e9:.1f} GB", flush=True)
        if it == 6:
            Path("gpurun_out").mkdir(exist_ok=True)
            Path(f"gpurun_out/timeline_{'_'.join(tier_set)}_p{pool}_c{cache}_r{ring}_z{zc}_s{split}_h{hbm}_u{hsplit}.json").write_text(json.dumps(tl))
    steady = phases[3:]
    out.append(dict(pool=pool, cache=cache, ring=ring, zero_copy=zc, d2h_split=split, hbm_retain=hbm, h2d_split=hsplit,
                    init_s=init_s,
                    ms=statistics.mean(p["ms"] for p in steady), phases=phases))
    w.close()
    del w
print(json.dumps([{k: v for k, v in o.items() if k != "phases"} for o in out], indent=1))
Path(os.environ.get("TFB_SWEEP_OUT", "gpurun_out/e2e_sweep.json")).write_text(json.dumps(out, indent=1))
shutil.rmtree(root, ignore_errors=True)
shutil.rmtree(remote_root, ignore_errors=True)
