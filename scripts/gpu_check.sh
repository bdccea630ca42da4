#!/bin/bash
# Build, GPU tests (optionally filtered), and a list of extra commands; logs under gpurun_out/.
set -u
mkdir -p gpurun_out
python -m paper_2509_02480_b200.build > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
make -s -C oracle >> gpurun_out/build.log 2>&1
if [ -n "${TESTS-1}" ]; then
timeout ${TEST_TIMEOUT:-1200} python -m pytest tests -m gpu -q -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/gpu_tests.log 2>&1
echo "pytest rc=$?"; tail -15 gpurun_out/gpu_tests.log
fi
i=0
while [ $# -gt 0 ]; do
  i=$((i+1)); echo "== cmd $i: $1"
  timeout ${CMD_TIMEOUT:-1200} bash -c "$1" > gpurun_out/cmd$i.log 2>&1; echo "rc=$?"; tail -${TAIL:-25} gpurun_out/cmd$i.log
  shift
done
