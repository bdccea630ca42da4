#!/bin/bash
# One GPU-box pass: build, gpu tests, smoke, a short bench. Logs under gpurun_out/.
set -u
mkdir -p gpurun_out
python -m paper_2509_02480_b200.build > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
make -s -C oracle >> gpurun_out/build.log 2>&1
timeout ${TEST_TIMEOUT:-1200} python -m pytest tests -m gpu -q ${PYTEST_ARGS:-} > gpurun_out/gpu_tests.log 2>&1
echo "pytest rc=$?"; tail -40 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -5 gpurun_out/smoke.log
if [ -n "${BENCH:-1}" ]; then
  timeout ${BENCH_TIMEOUT:-1500} python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err
  echo "bench rc=$?"; cat gpurun_out/bench.json; tail -20 gpurun_out/bench.err
fi
