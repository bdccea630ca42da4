"""Times the fused reduce + update kernel (tfg_adam_fused_multi) against the
single-source kernel on 100M-param subgroups: n gradient sources in local
HBM stand in for the n data-parallel ranks' contributions (on an NVSwitch
box n-1 of them are peer loads). Algorithmic bytes = 26 + 2n per param.

    python scripts/multi_sweep.py [n_params] [subgroups] [reps]
"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2509_02480_b200 import tierflow as tf  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
S = int(sys.argv[2]) if len(sys.argv) > 2 else 6
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
peak = json.loads(Path("MEASURED_PEAKS.json").read_text())["hbm_gbs"] if Path("MEASURED_PEAKS.json").exists() else 6650.0
dev = torch.device("cuda:0")
hy = tf.AdamHyper()
subs = []
for k in range(S):
    st = torch.empty(3 * n, device=dev)
    tf.synthetic_state(st[:n], st[n:2 * n], st[2 * n:], 42, k)
    subs.append((st, torch.empty(n, dtype=torch.int16, device=dev)))
srcs = []
for s in range(8):
    g = torch.empty(n, dtype=torch.int16, device=dev)
    tf.synthetic_grads(g, 42 + s, 0, 0)
    srcs.append(g)
torch.cuda.synchronize()
stream = torch.cuda.Stream()
out = {}
for label, nsrc in [("single", 1), ("multi1", 1), ("multi2", 2), ("multi3", 3), ("multi4", 4), ("multi8", 8)]:
    t = 1

    def launch(st, p16):
        if label == "single":
            tf.adam_fused(st[:n], st[n:2 * n], st[2 * n:], srcs[0], p16, t, hy, stream=stream)
        else:
            tf.adam_fused_multi(st[:n], st[n:2 * n], st[2 * n:], srcs[:nsrc], p16, t, hy, stream=stream)
    with torch.cuda.stream(stream):
        for st, p16 in subs:
            launch(st, p16)
            t += 1
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            for st, p16 in subs:
                launch(st, p16)
                t += 1
        b.record(stream)
    stream.synchronize()
    us = a.elapsed_time(b) * 1e3 / (reps * S)
    bpp = 28 if label == "single" else 26 + 2 * nsrc
    gbs = bpp * n / (us * 1e-6) / 1e9
    out[label] = {"sources": nsrc, "us_per_launch": round(us, 1), "alg_bytes_per_param": bpp, "GBs": round(gbs, 1),
                  "frac": round(gbs / peak, 4)}
    print(f"{label:7s} n={nsrc}: {us:8.1f} us  {gbs:7.1f} GB/s  {gbs / peak:.3f}", flush=True)
Path("gpurun_out").mkdir(exist_ok=True)
Path("gpurun_out/multi_sweep.json").write_text(json.dumps(out, indent=1))
