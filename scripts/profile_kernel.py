"""Launches the fused Adam kernel on 100M-param subgroups for ncu captures.

    ncu --set full -k regex:adam_fused -s 2 -c 1 -o gpurun_out/prof python scripts/profile_kernel.py
    python scripts/profile_kernel.py [n] [reps] [grad_kind] [sources] [gated]   (sources > 0: the
        n-source reduce + update form, tfg_adam_fused_multi, over `sources` local gradient buffers;
        gated = 1 (default): single-source launches behind a zero device gate, as the bench's device
        leg and the engine run them — the shipped staged kernel without the second non-finite count)
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2509_02480_b200 import tierflow as tf  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
gk = int(sys.argv[3]) if len(sys.argv) > 3 else 0
nsrc = int(sys.argv[4]) if len(sys.argv) > 4 else 0
gated = (int(sys.argv[5]) if len(sys.argv) > 5 else 1) != 0
dev = torch.device("cuda:0")
subs = []
for k in range(reps):
    st = torch.empty(3 * n, device=dev)
    g = torch.empty(n, dtype=torch.int16, device=dev)
    tf.synthetic_state(st[:n], st[n:2 * n], st[2 * n:], 42, k)
    tf.synthetic_grads(g, 42, k, 0, dtype=gk)
    subs.append((st, g, torch.empty(n, dtype=torch.int16, device=dev)))
extra = []
for s in range(1, nsrc):
    e = torch.empty(n, dtype=torch.int16, device=dev)
    tf.synthetic_grads(e, 43 + s, 0, 0, dtype=gk)
    extra.append(e)
gate = torch.zeros(1, dtype=torch.int64, device=dev) if gated else None
torch.cuda.synchronize()
for t, (st, g, p16) in enumerate(subs, start=1):
    if nsrc > 0:
        tf.adam_fused_multi(st[:n], st[n:2 * n], st[2 * n:], [g] + extra, p16, t, tf.AdamHyper(), gk, 0)
    else:
        tf.adam_fused(st[:n], st[n:2 * n], st[2 * n:], g, p16, t, tf.AdamHyper(), gk, 0, gate=gate)
torch.cuda.synchronize()
print("done")
