#!/bin/bash
# ncu evidence for the fused kernel: launch list of a short bench and --set full captures of the
# single-source kernel and of the 2- and 8-source reduce + update forms.
set -u
mkdir -p gpurun_out
python -m paper_2509_02480_b200.build > gpurun_out/build.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --skip-e2e --skip-cpu --skip-spill > gpurun_out/ncu_bench.log 2>&1
echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:adam_staged -s 2 -c 1 \
  -o gpurun_out/prof_adam -f python scripts/profile_kernel.py > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"; tail -3 gpurun_out/ncu_full.log
for k in ${MULTI:-2 8}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:adam_(staged|fused)" -s 2 -c 1 \
    -o gpurun_out/prof_multi$k -f python scripts/profile_kernel.py 100000000 4 0 $k > gpurun_out/ncu_multi$k.log 2>&1
  echo "multi$k rc=$?"
done
