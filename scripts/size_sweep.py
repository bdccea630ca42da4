"""fused-kernel throughput against subgroup size (64M .. 1B params
per launch), sources and state in HBM, CUDA events on the launching stream.

    python scripts/size_sweep.py
"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2509_02480_b200 import tierflow as tf  # noqa: E402

peak = bench.peaks()["hbm_gbs"]
out = {}
for n in (64_000_000, 100_000_000, 250_000_000, 500_000_000, 1_000_000_000):
    reps = max(2, 2_000_000_000 // n)
    st = torch.empty(3 * n, device="cuda")
    g = torch.empty(n, dtype=torch.int16, device="cuda")
    p16 = torch.empty(n, dtype=torch.int16, device="cuda")
    tf.synthetic_state(st[:n], st[n:2 * n], st[2 * n:], 42, 0)
    tf.synthetic_grads(g, 42, 0, 0)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for t in range(1, 3):
            tf.adam_fused(st[:n], st[n:2 * n], st[2 * n:], g, p16, t, tf.AdamHyper(), stream=s)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for t in range(3, 3 + reps):
            tf.adam_fused(st[:n], st[n:2 * n], st[2 * n:], g, p16, t, tf.AdamHyper(), stream=s)
        b.record(s)
    s.synchronize()
    us = a.elapsed_time(b) * 1e3 / reps
    gbs = 28 * n / (us * 1e-6) / 1e9
    out[n] = {"us_per_launch": round(us, 1), "GBs": round(gbs, 1), "frac": round(gbs / peak, 4)}
    print(f"{n/1e6:6.0f}M params: {us:9.1f} us  {gbs:7.1f} GB/s  {gbs / peak:.3f}", flush=True)
    del st, g, p16
    torch.cuda.empty_cache()
Path("gpurun_out").mkdir(exist_ok=True)
Path("gpurun_out/size_sweep.json").write_text(json.dumps(out, indent=1))
