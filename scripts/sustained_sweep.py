"""Kernel variants under sustained load (the bench's regime: 68 x 100M-param
launches per step, back to back, where the 1 kW power cap lowers SM clocks).
Variants are interleaved in rounds so clock drift affects them alike.

    python scripts/sustained_sweep.py [variants=0,26] [rounds=3] [steps=6]
"""
import json
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2509_02480_b200 import tierflow as tf  # noqa: E402

variants = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "0,26").split(",")]
if 67 in variants:  # it reads the state as tile-interleaved: it would corrupt the shared P || m || v buffers
    sys.exit("variant 67 changes the state layout: use scripts/layout_probe.py")
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 3
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 6
sizes = bench.subgroup_sizes(6_738_415_616, 100_000_000)
dev = torch.device("cuda:0")
stream = torch.cuda.Stream()
states, grads, p16s = [], [], []
with torch.cuda.stream(stream):
    for k, n in enumerate(sizes):
        st = torch.empty(3 * n, device=dev)
        g = torch.empty(n, dtype=torch.int16, device=dev)
        tf.synthetic_state(st[:n], st[n:2 * n], st[2 * n:], 42, k, stream=stream)
        tf.synthetic_grads(g, 42, k, 0, stream=stream)
        states.append(st)
        grads.append(g)
        p16s.append(torch.empty(n, dtype=torch.int16, device=dev))
stream.synchronize()
hy = tf.AdamHyper()
peak = bench.peaks()["hbm_gbs"]
res = {v: [] for v in variants}
t = 1
for r in range(rounds):
    for v in variants:
        with torch.cuda.stream(stream):
            for _ in range(2):  # warm
                for k, n in enumerate(sizes):
                    st = states[k]
                    tf.adam_fused_variant(v, st[:n], st[n:2 * n], st[2 * n:], grads[k], p16s[k], t, hy, stream=stream)
                t += 1
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with bench.ClockSampler(0) as clk:
                a.record(stream)
                for _ in range(steps):
                    for k, n in enumerate(sizes):
                        st = states[k]
                        tf.adam_fused_variant(v, st[:n], st[n:2 * n], st[2 * n:], grads[k], p16s[k], t, hy,
                                              stream=stream)
                    t += 1
                b.record(stream)
                stream.synchronize()
        ms = a.elapsed_time(b) / steps
        gbs = 28 * sum(sizes) / (ms / 1e3) / 1e9
        c = clk.summary()
        res[v].append({"ms_per_step": round(ms, 2), "GBs": round(gbs, 1), "frac": round(gbs / peak, 4),
                       "sm_mhz": c["sm_mhz"], "reasons": c["reasons"]})
        print(f"round {r} variant {v}: {ms:.2f} ms/step {gbs:.1f} GB/s {gbs / peak:.3f} sm {c['sm_mhz']} {c['reasons']}",
              flush=True)
summary = {v: {"mean_frac": round(statistics.mean(x["frac"] for x in res[v]), 4), "runs": res[v]} for v in variants}
print(json.dumps({v: s["mean_frac"] for v, s in summary.items()}))
Path("gpurun_out").mkdir(exist_ok=True)
Path("gpurun_out/sustained_sweep.json").write_text(json.dumps(summary, indent=1))
