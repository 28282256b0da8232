#!/bin/bash
# First-pass GPU check: debug build (mbarrier waits trap instead of hanging),
# smoke, then the GPU parity suite.  Output under gpurun_out/.
set -u
mkdir -p gpurun_out
export RELAX_Q4_DEBUG=${RELAX_Q4_DEBUG:-1}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD_FAIL; tail -30 gpurun_out/build.log; exit 1; }
timeout 180 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?"; tail -20 gpurun_out/smoke.log
timeout ${PYTEST_TIMEOUT:-1200} python -m pytest tests -m gpu -x -q --timeout 300 ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -40 gpurun_out/pytest_gpu.log
