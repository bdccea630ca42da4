#!/bin/bash
# Kernel-variant sweep + e2e pipeline sweep + box memory inventory. Logs under gpurun_out/.
set -u
mkdir -p gpurun_out
python -m paper_2509_02480_b200.build > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
{ free -g; nproc; grep -E "MemTotal|MemAvailable|Hugepagesize" /proc/meminfo; nvidia-smi --query-gpu=memory.total,clocks.max.sm,power.limit --format=csv; df -h "$GRAFT_REPO_ROOT" /tmp /dev/shm; lsblk -o NAME,SIZE,TYPE,ROTA,MOUNTPOINT 2>/dev/null | head -20; } > gpurun_out/box.txt 2>&1
if [ -n "${KSWEEP:-1}" ]; then
timeout 900 python scripts/kernel_sweep.py > gpurun_out/kernel_sweep.log 2>&1; echo "kernel sweep rc=$?"; grep variant gpurun_out/kernel_sweep.log; grep -A3 div_selftest gpurun_out/kernel_sweep.log | head -5
fi
if [ -n "${E2E_CONFIGS:-}" ]; then
timeout 1500 python scripts/e2e_sweep.py 6738415616 $E2E_CONFIGS > gpurun_out/e2e_sweep.log 2>&1; echo "e2e sweep rc=$?"; tail -40 gpurun_out/e2e_sweep.log
fi
if [ -n "${SPILL_CONFIGS:-}" ]; then
TFB_TIERS=nvme,remote TFB_SWEEP_OUT=gpurun_out/e2e_spill.json timeout 1500 python scripts/e2e_sweep.py ${SPILL_TOTAL:-2000000000} $SPILL_CONFIGS > gpurun_out/e2e_spill.log 2>&1; echo "spill sweep rc=$?"; grep -E "probe|phase" gpurun_out/e2e_spill.log | tail -30
fi
cat gpurun_out/box.txt
