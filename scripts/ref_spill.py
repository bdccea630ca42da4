"""The reference CPU engine on the spill shape of bench.py's `spill` leg, for
a like-for-like comparison: 12 subgroups x 100M params on a local and a
"remote" directory tier on the box's disk, pool 8 (the reference's C =
pool - 3 = 5), all host threads, 3 iterations (the last 2 timed).

    python scripts/ref_spill.py [subgroups=12] [sub=100000000]
"""
import json
import os
import shutil
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import oracle  # noqa: E402  (the reference engine, oracle/_ref)

M = int(sys.argv[1]) if len(sys.argv) > 1 else 12
sub = int(sys.argv[2]) if len(sys.argv) > 2 else 100_000_000
root = ROOT / "gpurun_out" / "ref_spill_tiers"
shutil.rmtree(root, ignore_errors=True)
root.mkdir(parents=True)
# rates as the B200 engine's probe measured the box's disk (both roots share it)
tiers = [dict(kind=0, root=str(root / "nvme"), read_bps=5.2e9, write_bps=5.1e9, io_parallelism=4),
         dict(kind=1, root=str(root / "remote"), read_bps=5.2e9, write_bps=5.1e9, io_parallelism=4)]
threads = os.cpu_count() or 1
res = oracle.run_ref_engine([sub] * M, tiers, pool_slots=8, update_threads=threads, lock_dir=str(root / "locks"),
                            seed=42, iterations=3, want_states=False, events_cap=1)
shutil.rmtree(root, ignore_errors=True)
its = res["iters"]
for i, it in enumerate(its):
    print(f"iteration {i}: update {it['update_seconds']:.2f} s, hits {it['cache_hits']}, "
          f"alloc {it['flush_allocation']}", flush=True)
timed = its[1:]
out = {"subgroups": M, "params_per_subgroup": sub, "threads": threads,
       "update_s": statistics.mean(t["update_seconds"] for t in timed),
       "params_per_s": M * sub / statistics.mean(t["update_seconds"] for t in timed),
       "iters": its}
print(json.dumps({k: v for k, v in out.items() if k != "iters"}))
Path("gpurun_out/ref_spill.json").write_text(json.dumps(out, indent=1))
