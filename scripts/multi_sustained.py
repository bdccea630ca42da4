"""The fused reduce + update under the bench's sustained load: the staged
n-source kernel (2, 4, 8 sources) against the register n-source kernel,
interleaved rounds, n gradient sources in local HBM standing in for
the ranks' NVLink-mapped contributions. Algorithmic bytes 26 + 2n per param.

    python scripts/multi_sustained.py [sources=2,4,8] [rounds=3] [steps=4] [subgroups=48]
"""
import json
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2509_02480_b200 import tierflow as tf  # noqa: E402

nsrcs = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "2,4,8").split(",")]
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 3
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
M = int(sys.argv[4]) if len(sys.argv) > 4 else 48
n = 100_000_000
dev = torch.device("cuda:0")
stream = torch.cuda.Stream()
states = []
for k in range(M):
    st = torch.empty(3 * n, device=dev)
    tf.synthetic_state(st[:n], st[n:2 * n], st[2 * n:], 42, k, stream=stream)
    states.append(st)
srcs = []
for s in range(max(nsrcs)):
    g = torch.empty(n, dtype=torch.int16, device=dev)
    tf.synthetic_grads(g, 43 + s, 0, 0, stream=stream)
    srcs.append(g)
p16 = torch.empty(n, dtype=torch.int16, device=dev)
stream.synchronize()
peak = bench.peaks()["hbm_gbs"]
hy = tf.AdamHyper()
res = {}
t = 1
for r in range(rounds):
    for ns in nsrcs:
        for form in (0, 1):
            def step():
                for st in states:
                    tf.adam_fused_multi_variant(form, st[:n], st[n:2 * n], st[2 * n:], srcs[:ns], p16, t, hy,
                                                stream=stream)
            with torch.cuda.stream(stream):
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
            gbs = (26 + 2 * ns) * M * n / (ms / 1e3) / 1e9
            key = f"n{ns}_{'staged' if form == 0 else 'register'}"
            res.setdefault(key, []).append(round(gbs / peak, 4))
            print(f"round {r} {key}: {ms:.2f} ms/step {gbs:.1f} GB/s {gbs / peak:.3f} sm {clk.summary()['sm_mhz']}",
                  flush=True)
summary = {k: round(statistics.mean(v), 4) for k, v in res.items()}
print(json.dumps(summary))
Path("gpurun_out").mkdir(exist_ok=True)
Path("gpurun_out/multi_sustained.json").write_text(json.dumps({"mean_frac": summary, "runs": res}, indent=1))
