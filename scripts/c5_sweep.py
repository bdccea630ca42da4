"""SURVEY §8 C5 (BASELINE configs[4]): subgroup-size x tier-mix sweep of the
update phase through the engine's C ABI (run_update), with the reference CPU
engine (oracle/_ref) timed beside each subgroup size on the host's cores.

    python scripts/c5_sweep.py [--sizes 64e6,100e6,250e6,500e6,1e9]
                               [--mixes dram,dram_nvme,spill] [--steps 3] [--warmup 4]

Tier mixes (one B200, this host):
  dram       every subgroup on the pinned host-DRAM tier (PCIe-bound)
  dram_nvme  host DRAM + a local O_DIRECT directory tier, Eq. 1 over both (C2's mix)
  spill      host DRAM capped at 2 subgroups, the rest on local + "remote"
             directory tiers sharing one device semaphore (C4's mix)
Each point keeps ~40% of its subgroups in the HBM cache (50% for spill, as
the bench's C4 sample); sizes are bounded by host memory and disk.
Writes gpurun_out/c5_sweep.json.
"""
import argparse
import json
import os
import shutil
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402

GB = 1e9


def point(tf, sub, mix, steps, warmup, root):
    import torch
    dev = torch.cuda.current_device()
    state = 12 * sub
    if mix == "spill":
        root.parent.mkdir(parents=True, exist_ok=True)
        free = shutil.disk_usage(root.parent).free
        M = int(max(3, min(36, round(2.4e9 / sub), 0.4 * free // (state + 4096))))
        C, dram_cap = M // 2, 2
    else:
        M = max(3, round(6.4e9 / sub))
        C, dram_cap = int(0.4 * M), 0
    pool = int(max(4, min(16, 24 * GB // state)))
    ring = int(max(2, min(12, 24 * GB // state)))
    sizes = [sub] * M
    shutil.rmtree(root, ignore_errors=True)
    (root / "nvme").mkdir(parents=True)
    (root / "remote").mkdir(parents=True)
    pcie = bench.pcie_probe()
    block = 4096 * ((32 + state + 4095) // 4096)
    dram_bw = min(pcie["h2d"], pcie["d2h"])
    tiers = [tf.Tier(tf.TierSpec(0, tf.TierKind.host_dram, "dram", dram_bw, dram_bw,
                                 capacity_bytes=dram_cap * block if dram_cap else 0))]
    if mix in ("dram_nvme", "spill"):
        tiers.append(tf.Tier(tf.TierSpec(1, tf.TierKind.local_dir, str(root / "nvme"), 0.0, 0.0, io_parallelism=4,
                                         lock_device=1)))
    if mix == "spill":
        tiers.append(tf.Tier(tf.TierSpec(2, tf.TierKind.remote_dir, str(root / "remote"), 0.0, 0.0,
                                         io_parallelism=4, lock_device=1)))
    probes = {t.id(): t.probe_bandwidth(1 << 30, 3) for t in tiers[1:]}
    trace = tf.EventTrace()
    opt = tf.ScheduleOptions(pool_slots=pool, cache_slots=C, lock_dir=str(root / "locks"))
    t0 = time.time()
    w = tf.OffloadWorker(0, tiers, opt, tf.AdamHyper(), trace, tf.DeviceOptions(dev, 0, 0, ring, 0, 1, 2))
    for k in range(M):
        w.add_subgroup(k, sub)
    w.init_and_flush_all(42)
    init_s = time.time() - t0
    src = tf.SyntheticGradSource(42)
    phases = bench.run_phases(w, 1, 0, warmup, steps, lambda it: w.run_backward_sim(it, src, 1), f"{mix} {sub:.0e}")
    rl = bench.pipeline_roofline(phases, pcie, probes)
    w.close()
    del w
    shutil.rmtree(root, ignore_errors=True)
    ms = statistics.mean(p[0] for p in phases)
    return dict(subgroup_params=sub, mix=mix, subgroups=M, retained_hbm=C, pool=pool, ring=ring,
                dram_cap_subgroups=dram_cap or None, ms_per_phase=round(ms, 1),
                params_per_s=M * sub / (ms / 1e3), bound_ms=round(rl["bound_s"] * 1e3, 1),
                pipeline_frac=round(rl["bound_s"] * 1e3 / ms, 4), pcie_bound_ms=round(rl["pcie_s"] * 1e3, 1),
                tier_bound_ms=round(rl["tier_s"] * 1e3, 1), per_tier=rl["per_tier"],
                flush_allocation=phases[-1][1].flush_allocation,
                hits=statistics.mean(p[1].cache_hits for p in phases), init_s=round(init_s, 1),
                pcie_gbs={k: round(v / GB, 1) for k, v in pcie.items()})


def reference_point(sub, root):
    """The reference engine on 2 subgroups of this size (C = 1, pool 4),
    [mem_throttled as DRAM, local_dir], all host threads; 1 timed phase."""
    import oracle
    threads = os.cpu_count() or 1
    shutil.rmtree(root, ignore_errors=True)
    root.mkdir(parents=True)
    tiers = [dict(kind=2, read_bps=50e9, write_bps=50e9), dict(kind=0, root=str(root / "nvme"), io_parallelism=4)]
    res = oracle.run_ref_engine([sub] * 2, tiers, pool_slots=4, cache_slots=1, update_threads=threads,
                                lock_dir=str(root / "locks"), seed=42, iterations=2, want_states=False, events_cap=1,
                                backward_once=True)
    shutil.rmtree(root, ignore_errors=True)
    it = res["iters"][-1]
    return dict(subgroup_params=sub, params_per_s=it["params_updated"] / it["update_seconds"], cores=threads,
                sample="reference OffloadWorker::run_update, 2 subgroups, C=1, pool 4, "
                       "[mem_throttled 50 GB/s, local_dir], 1 timed of 2 phases")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="64e6,100e6,250e6,500e6,1e9")
    ap.add_argument("--mixes", default="dram,dram_nvme,spill")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=4)
    ap.add_argument("--skip-reference", action="store_true")
    a = ap.parse_args()
    from paper_2509_02480_b200 import tierflow as tf
    sizes = [int(float(x)) for x in a.sizes.split(",")]
    root = ROOT / "gpurun_out" / "c5_tiers"
    out = {"points": [], "reference": []}
    for sub in sizes:
        for mix in a.mixes.split(","):
            try:
                r = point(tf, sub, mix, a.steps, a.warmup, root)
            except Exception as exc:  # noqa: BLE001 - recorded, the sweep goes on
                r = dict(subgroup_params=sub, mix=mix, error=f"{type(exc).__name__}: {exc}")
            print(json.dumps(r), flush=True)
            out["points"].append(r)
            Path("gpurun_out/c5_sweep.json").write_text(json.dumps(out, indent=1))
    if not a.skip_reference:
        for sub in sizes:
            try:
                r = reference_point(sub, root)
            except Exception as exc:  # noqa: BLE001
                r = dict(subgroup_params=sub, error=f"{type(exc).__name__}: {exc}")
            print(json.dumps(r), flush=True)
            out["reference"].append(r)
            Path("gpurun_out/c5_sweep.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
