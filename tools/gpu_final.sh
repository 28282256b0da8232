#!/bin/bash
# Round-end style pass: build, GPU tests, bench (7B decode, prefill n=512, 13B), launch list, ncu of top kernels.
set -u
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD_FAIL; exit 1; }
timeout 180 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
if [ "${SKIP_TESTS:-0}" != "1" ]; then
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
fi
timeout 600 python bench.py > gpurun_out/bench_7b.json 2> gpurun_out/bench_7b.err; echo "bench 7b rc=$?"; cat gpurun_out/bench_7b.json
timeout 600 python bench.py --workload llama2-7b-prefill --n 512 --no-cpu-baseline > gpurun_out/bench_7b_prefill.json 2> gpurun_out/bench_7b_prefill.err; echo "bench prefill rc=$?"
timeout 600 python bench.py --workload llama2-13b-decode --no-cpu-baseline > gpurun_out/bench_13b.json 2> gpurun_out/bench_13b.err; echo "bench 13b rc=$?"
timeout 600 python bench.py --impl reference --steps 2 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "bench ref rc=$?"; cat gpurun_out/bench_ref.json
if [ "${NCU:-1}" = "1" ]; then
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ll_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 1000 -c 300 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_ll.log 2>&1; echo "launch list rc=$?"
timeout 100 python tools/prof_one.py 4096 11008 1 auto 5 > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv -s 2 -c 1 -o gpurun_out/prof_gemv_4096x11008_n1 python tools/prof_one.py 4096 11008 1 auto 5 > gpurun_out/ncu1.log 2>&1; echo "ncu gemv rc=$?"
timeout 100 python tools/prof_one.py 4096 11008 512 auto 5 > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_q4 -s 2 -c 1 -o gpurun_out/prof_tc_4096x11008_n512 python tools/prof_one.py 4096 11008 512 auto 5 > gpurun_out/ncu2.log 2>&1; echo "ncu tc rc=$?"
fi
