"""The paper's ablation ladder (reference acceptance
criterion 10) on the B200 engine at the Llama-2-7B shape: the ZeRO-3
baseline flow (fp32 gradients through storage, ascending order only, one
tier) and then each MLP-Offload technique switched on, through host DRAM +
an O_DIRECT directory tier. Reports the backward-side gradient flush (the
baseline's extra storage traffic), the update phase and their sum.

    python scripts/ablation_sweep.py [total_params] [phases]

Each rung runs in its own process (pinned host memory is returned to the OS
at process exit; the GPU boxes' sandbox does not always reclaim it earlier).
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
phases = int(sys.argv[2]) if len(sys.argv) > 2 else 6
sub = 100_000_000
sizes = [min(sub, total - k * sub) for k in range((total + sub - 1) // sub)]
root = ROOT / "gpurun_out" / "ablation_tiers"
# (name, caching, skip_gradients, atomic_rw, multi_path, pool, cache, hbm_retain)
M = len(sizes)
c_host, c_hbm = round(13 * M / 68), round(29 * M / 68)  # the bench's retained fractions at the 7B shape
ladder = [
    ("zero3_baseline", False, False, False, False, 16, 0, 0),
    ("+caching", True, False, False, False, 16, c_host, 0),
    ("+skip_gradients", True, True, False, False, 16, c_host, 0),
    ("+atomic_rw", True, True, True, False, 16, c_host, 0),
    ("+multi_path (MLP-Offload)", True, True, True, True, 16, c_host, 0),
    ("+HBM cache (B200)", True, True, True, True, 16, c_hbm, 2),
    ("+two-level HBM + host (B200)", True, True, True, True, 16, c_hbm + c_host, 2),
]
import os
import subprocess

if len(sys.argv) > 3:  # child: one rung
    ladder = [ladder[int(sys.argv[3])]]
else:
    out = []
    for i in range(len(ladder)):
        r = subprocess.run([sys.executable, __file__, str(total), str(phases), str(i)], capture_output=True, text=True)
        sys.stdout.write(r.stdout)
        sys.stderr.write(r.stderr[-2000:])
        try:
            out.append(json.loads(r.stdout.strip().splitlines()[-1]))
        except (IndexError, json.JSONDecodeError):
            out.append({"config": ladder[i][0], "error": r.stderr.strip().splitlines()[-1] if r.stderr else "?"})
    base = out[0]
    for r in out:
        if "update_s" in r and "update_s" in base:
            r["update_speedup_vs_zero3"] = base["update_s"] / r["update_s"]
            r["iteration_speedup_vs_zero3"] = base["iteration_s"] / r["iteration_s"]
    print(json.dumps(out, indent=1))
    Path(os.environ.get("TFB_SWEEP_OUT", "gpurun_out/ablation_sweep.json")).write_text(json.dumps(out, indent=1))
    sys.exit(0)

for name, caching, skip, atomic, multi, pool, cache, hbm in ladder:
    shutil.rmtree(root, ignore_errors=True)
    if os.environ.get("TFB_TIERS", "dram,nvme") == "nvme,remote":  # disk-bound: the paper's NVMe + PFS setting
        t0_ = tf.Tier(tf.TierSpec(0, tf.TierKind.local_dir, str(root / "nvme"), 0, 0, io_parallelism=4,
                                  lock_device=1))
        t1_ = tf.Tier(tf.TierSpec(1, tf.TierKind.remote_dir, str(root / "remote"), 0, 0, io_parallelism=4,
                                  lock_device=1))
        t0_.probe_bandwidth(1 << 30, 3)
    else:
        t0_ = tf.Tier(tf.TierSpec(0, tf.TierKind.host_dram, "dram", 50e9, 50e9))
        t1_ = tf.Tier(tf.TierSpec(1, tf.TierKind.local_dir, str(root / "nvme"), 0, 0, io_parallelism=4))
    t1_.probe_bandwidth(1 << 30, 3)
    dram, nvme = t0_, t1_
    opt = tf.ScheduleOptions(pool_slots=pool, cache_slots=cache, enable_caching=caching, skip_gradients=skip,
                             atomic_rw=atomic, multi_path=multi, lock_dir=str(root / "locks"))
    hbm_slots = c_hbm if name.startswith("+two-level") else 0
    w = tf.OffloadWorker(0, [dram, nvme], opt, tf.AdamHyper(), tf.EventTrace(),
                         tf.DeviceOptions(0, 0, 0, 12, 0, 1, hbm, 1, hbm_slots))
    for k, n in enumerate(sizes):
        w.add_subgroup(k, n)
    w.init_and_flush_all(42)
    rows = []
    for it in range(phases):
        t0 = time.perf_counter()
        w.run_backward_sim(it, tf.SyntheticGradSource(42))
        torch.cuda.synchronize()
        bwd = time.perf_counter() - t0
        t0 = time.perf_counter()
        st = w.run_update(it)
        upd = time.perf_counter() - t0
        rows.append(dict(backward_s=bwd, update_s=upd, hits=st.cache_hits, alloc=st.flush_allocation,
                         h2d=st.h2d_bytes, d2h=st.d2h_bytes))
        print(f"{name:28s} phase {it}: backward {bwd*1e3:7.0f} ms update {upd*1e3:7.0f} ms hits {st.cache_hits:2d} "
              f"alloc {st.flush_allocation} h2d {st.h2d_bytes/1e9:.1f} GB", flush=True)
    w.close()
    del w
    steady = rows[2:]
    r = dict(config=name, backward_s=statistics.mean(x["backward_s"] for x in steady),
             update_s=statistics.mean(x["update_s"] for x in steady), hits=steady[-1]["hits"],
             alloc=steady[-1]["alloc"], h2d_gb=steady[-1]["h2d"] / 1e9)
    r["iteration_s"] = r["backward_s"] + r["update_s"]
    shutil.rmtree(root, ignore_errors=True)
    print(json.dumps(r), flush=True)
