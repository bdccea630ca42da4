"""Layout experiment: the staged kernel on P || m || v (shipped, variant 55)
vs the tile-interleaved state layout (tuning variant 67: per 1024-param tile
[P | m | v] contiguous), each on its own zero-initialised state (valid for
both layouts), interleaved rounds under sustained load.

    python scripts/layout_probe.py [subgroups=34] [rounds=4] [steps=6]
"""
import json
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2509_02480_b200 import tierflow as tf  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 34
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 4
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 6
n = 100_000_000 // 1024 * 1024
dev = torch.device("cuda:0")
stream = torch.cuda.Stream()
grads = []
for k in range(M):
    g = torch.empty(n, dtype=torch.int16, device=dev)
    tf.synthetic_grads(g, 42, k, 0, stream=stream)
    grads.append(g)
sets = {v: [torch.zeros(3 * n, device=dev) for _ in range(M)] for v in (55, 67)}
p16 = torch.empty(n, dtype=torch.int16, device=dev)
stream.synchronize()
hy = tf.AdamHyper()
peak = bench.peaks()["hbm_gbs"]
res = {v: [] for v in sets}
t = 1
for r in range(rounds):
    for v, states in sets.items():
        with torch.cuda.stream(stream):
            def step():
                for k in range(M):
                    st = states[k]
                    tf.adam_fused_variant(v, st[:n], st[n:2 * n], st[2 * n:], grads[k], p16, t, hy, stream=stream)
            step()
            step()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with bench.ClockSampler(0) as clk:
                a.record(stream)
                for _ in range(steps):
                    step()
                b.record(stream)
                stream.synchronize()
        t += 1
        ms = a.elapsed_time(b) / steps
        gbs = 28 * M * n / (ms / 1e3) / 1e9
        c = clk.summary()
        res[v].append(round(gbs / peak, 4))
        print(f"round {r} variant {v}: {ms:.2f} ms/step {gbs:.1f} GB/s {gbs / peak:.3f} sm {c['sm_mhz']}", flush=True)
        # sanity: the state stays finite
        assert all(bool(torch.isfinite(s[:1 << 20]).all()) for s in states[:2]), v
summary = {v: round(statistics.mean(x), 4) for v, x in res.items()}
print(json.dumps(summary))
Path("gpurun_out").mkdir(exist_ok=True)
Path("gpurun_out/layout_probe.json").write_text(json.dumps({"mean_frac": summary, "runs": res}, indent=1))
