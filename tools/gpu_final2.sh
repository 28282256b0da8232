#!/bin/bash
# End-of-round re-check on the final code: build, smoke, pytest -m gpu, bench lines (decode, prefill, 70B prefill)
set -u
O=gpurun_out/fin4; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo BUILD_FAIL; exit 1; }
timeout 180 python __graft_entry__.py --smoke > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 2000 python -m pytest tests -m gpu -q --timeout 600 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
b() { tag=$1; shift; timeout 900 python bench.py "$@" > $O/bench_$tag.json 2> $O/bench_$tag.err; echo "bench $tag rc=$? $(python -c "import json; d=json.load(open('$O/bench_$tag.json')); print(d['value'], d['hbm_gbs'], d['tflops'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>&1 | tail -1)"; }
b 7b_decode
b 7b_prefill_n512 --workload llama2-7b-prefill --n 512 --no-cpu-baseline
b 7b_prefill_n4096 --workload llama2-7b-prefill --n 4096 --steps 5 --no-cpu-baseline
b 13b_prefill_n512 --workload llama2-13b-prefill --n 512 --no-cpu-baseline
b 70b_prefill_n512 --workload llama2-70b-prefill --n 512 --steps 5 --no-cpu-baseline
b 70b_prefill_n4096 --workload llama2-70b-prefill --n 4096 --steps 3 --warmup 3 --no-cpu-baseline
b 7b_decode_batch64 --n 64 --no-cpu-baseline
b 70b_decode --workload llama2-70b-decode --no-cpu-baseline
b 7b_decode_batch8 --n 8 --no-cpu-baseline
timeout 600 python bench.py --impl reference --steps 2 > $O/bench_reference.json 2> $O/bench_reference.err; echo "reference rc=$? $(cut -c1-160 $O/bench_reference.json)"
