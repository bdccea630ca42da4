#!/bin/bash
# compute-sanitizer passes: memcheck over the engine smoke run (pipeline, HBM
# cache, directory tier) and over the fused reduce + update kernel; racecheck
# and synccheck over the shared-memory kernel variants (TMA, cp.async).
set -u
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
python -m paper_2509_02480_b200.build > gpurun_out/build.log 2>&1 || exit 1
make -s -C oracle >> gpurun_out/build.log 2>&1
timeout 900 $CS --tool memcheck --leak-check full --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_memcheck_smoke.log 2>&1
echo "memcheck smoke rc=$?"; tail -3 gpurun_out/san_memcheck_smoke.log
cat > /tmp/san_engine.py <<'PY'
# HBM cache mode (write-back lane) and the ZeRO-3 baseline flow (gradient stages), 3 phases each
import sys, tempfile, os
sys.path.insert(0, ".")
from paper_2509_02480_b200 import tierflow as tf
for hbm, skip in ((2, True), (0, False)):
    with tempfile.TemporaryDirectory() as d:
        tiers = [tf.Tier(tf.TierSpec(0, tf.TierKind.host_dram, "dram", 20e9, 20e9)),
                 tf.Tier(tf.TierSpec(1, tf.TierKind.local_dir, os.path.join(d, "n"), 2e9, 2e9))]
        w = tf.OffloadWorker(0, tiers, tf.ScheduleOptions(pool_slots=4, cache_slots=2, lock_dir=os.path.join(d, "l"),
                                                          skip_gradients=skip),
                             tf.AdamHyper(), tf.EventTrace(), tf.DeviceOptions(0, 0, 0, 2, 0, 1, hbm))
        w.set_fixed_ratio([1.0, 1.0])
        for i in range(5):
            w.add_subgroup(i, 40_000 + 3 * i)
        w.init_and_flush_all(1)
        for it in range(3):
            w.run_backward_sim(it, tf.SyntheticGradSource(1))
            w.run_update(it)
        w.close()
        del w, tiers
print("engine modes ok", tf.host_blocks_live(), tf.host_block_free_failures())
PY
timeout 900 $CS --tool memcheck --error-exitcode 9 python /tmp/san_engine.py > gpurun_out/san_memcheck_engine.log 2>&1
echo "memcheck engine modes rc=$?"; tail -3 gpurun_out/san_memcheck_engine.log
cat > /tmp/san_kernels.py <<'PY'
import sys
sys.path.insert(0, ".")
import torch
from paper_2509_02480_b200 import tierflow as tf
# a multiple of the TMA tile so every variant takes its main path (argv[2]: another size, e.g. with a tail)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1_003_520
variants = [int(v) for v in sys.argv[1].split(",")]
for v in variants:
    # P, m, v in separate (aligned) allocations: any n keeps every stream 16-byte aligned
    P, M, V = (torch.empty(n, device="cuda") for _ in range(3)); g = torch.empty(n, dtype=torch.int16, device="cuda")
    tf.synthetic_state(P, M, V, 1, 0); tf.synthetic_grads(g, 1, 0, 0)
    p16 = torch.empty(n, dtype=torch.int16, device="cuda")
    tf.adam_fused_variant(v, P, M, V, g, p16, 1, tf.AdamHyper())
    torch.cuda.synchronize()
st = torch.empty(3 * n, device="cuda")
srcs = [torch.empty(n, dtype=torch.int16, device="cuda") for _ in range(8)]
for s_ in srcs: tf.synthetic_grads(s_, 2, 0, 0)
tf.adam_fused_multi(st[:n], st[n:2*n], st[2*n:], srcs[:3], p16, 2, tf.AdamHyper())  # register n-source form
P, M, V = (torch.empty(n, device="cuda") for _ in range(3)); tf.synthetic_state(P, M, V, 1, 0)
tf.adam_fused_multi(P, M, V, srcs, p16, 3, tf.AdamHyper())  # 8 sources: the staged n-source kernel
torch.cuda.synchronize()
print("kernels ok")
PY
timeout 900 $CS --tool memcheck --error-exitcode 9 python /tmp/san_kernels.py 0,1,12,16,32,36,38,54,55 > gpurun_out/san_memcheck_kernels.log 2>&1
echo "memcheck kernels rc=$?"; tail -3 gpurun_out/san_memcheck_kernels.log
# the shipped staged kernel with a tail (n % 1024 = 3: one partial tile's quads and scalars in the last CTA)
timeout 900 $CS --tool memcheck --error-exitcode 9 python /tmp/san_kernels.py 0,55 1003523 > gpurun_out/san_memcheck_tail.log 2>&1
echo "memcheck staged tail rc=$?"; tail -3 gpurun_out/san_memcheck_tail.log
# a partial 2048-param tile of 577 params (n % 4 = 1) for the shipped 2 x 512 shape
timeout 900 $CS --tool memcheck --error-exitcode 9 python /tmp/san_kernels.py 0,70 1000001 > gpurun_out/san_memcheck_tail2.log 2>&1
echo "memcheck staged tail2 rc=$?"; tail -3 gpurun_out/san_memcheck_tail2.log
timeout 900 $CS --tool racecheck --error-exitcode 9 python /tmp/san_kernels.py 0,12,13,16,32,33,36,38,39,55,70 > gpurun_out/san_racecheck.log 2>&1
echo "racecheck rc=$?"; tail -3 gpurun_out/san_racecheck.log
timeout 900 $CS --tool synccheck --error-exitcode 9 python /tmp/san_kernels.py 0,12,16,32,36,38,55,70 > gpurun_out/san_synccheck.log 2>&1
echo "synccheck rc=$?"; tail -3 gpurun_out/san_synccheck.log
