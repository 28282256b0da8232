#!/bin/bash
# Iteration pass: tests, bench variants, sweep.
set -u
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD_FAIL; tail -20 gpurun_out/build.log; exit 1; }
if [ "${SKIP_TESTS:-0}" != "1" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x --timeout 300 ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1
  echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
fi
i=0
for v in "${BENCHES[@]:-}"; do
  i=$((i+1))
  env $v timeout 600 python bench.py --no-cpu-baseline ${BENCH_EXTRA:-} > gpurun_out/bench_$i.json 2> gpurun_out/bench_$i.err
  echo "bench[$v] rc=$? $(python -c "import json,sys;d=json.load(open('gpurun_out/bench_$i.json'));print(d['value'],d['unit'],d['hbm_gbs'],'GB/s',d['ms_per_step'],'ms')" 2>/dev/null)"
done
if [ -n "${SWEEP_ARGS:-}" ]; then
  rm -f gpurun_out/sweep.jsonl
  timeout 900 python tools/sweep.py $SWEEP_ARGS > gpurun_out/sweep.log 2>&1; echo "sweep rc=$?"
fi
