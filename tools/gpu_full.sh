#!/bin/bash
# Full GPU pass: build, smoke, whole -m gpu suite, bench lines.
set -u
O=gpurun_out/full; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo BUILD_FAIL; tail $O/build.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 $O/pytest_gpu.log
b() { tag=$1; shift; timeout 900 python bench.py "$@" > $O/bench_$tag.json 2> $O/bench_$tag.err; echo "bench $tag rc=$? $(python -c "import json; d=json.load(open('$O/bench_$tag.json')); print(d['value'], d['hbm_gbs'], d['tflops'], d['roofline']['frac'], d['e2e']['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>&1 | tail -1)"; }
b 7b_decode
b 7b_decode_fused --fused --no-cpu-baseline
b 7b_n4 --n 4 --no-cpu-baseline
b 7b_n8 --n 8 --no-cpu-baseline
b 7b_fused_n8 --fused --n 8 --no-cpu-baseline
b 7b_n32 --n 32 --no-cpu-baseline
b 7b_prefill_n512 --workload llama2-7b-prefill --n 512 --no-cpu-baseline
b 7b_prefill_n4096 --workload llama2-7b-prefill --n 4096 --steps 5 --no-cpu-baseline
