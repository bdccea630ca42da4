"""Launches one kernel-sweep variant on 100M-param subgroups (for ncu).

    ncu --set full -k regex:adam -s 2 -c 1 -o gpurun_out/prof_v33 python scripts/profile_variant.py 33
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2509_02480_b200 import tierflow as tf  # noqa: E402

v = int(sys.argv[1])
n = 100_000_000
dev = torch.device("cuda:0")
subs = []
for k in range(4):
    st = torch.empty(3 * n, device=dev)
    g = torch.empty(n, dtype=torch.int16, device=dev)
    tf.synthetic_state(st[:n], st[n:2 * n], st[2 * n:], 42, k)
    tf.synthetic_grads(g, 42, k, 0)
    subs.append((st, g, torch.empty(n, dtype=torch.int16, device=dev)))
torch.cuda.synchronize()
for t, (st, g, p16) in enumerate(subs, start=1):
    tf.adam_fused_variant(v, st[:n], st[n:2 * n], st[2 * n:], g, p16, t, tf.AdamHyper())
torch.cuda.synchronize()
print("done")
