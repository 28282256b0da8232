#!/bin/bash
set -u
O=gpurun_out/sn5; mkdir -p $O
python -m paper_2311_02103_b200.build > $O/build.log 2>&1 || { echo BUILD_FAIL; tail -5 $O/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_repack.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest repack rc=$?"; tail -2 $O/pytest.log
b() { tag=$1; shift; timeout 900 python bench.py "$@" > $O/bench_$tag.json 2> $O/bench_$tag.err; echo "bench $tag rc=$? $(python -c "import json; d=json.load(open('$O/bench_$tag.json')); print(d['value'], d['hbm_gbs'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>&1 | tail -1)"; }
b 7b_n3 --n 3 --no-cpu-baseline
b 7b_n4 --n 4 --no-cpu-baseline
b 7b_n8 --n 8 --no-cpu-baseline
b 7b_fused_n8 --fused --n 8 --no-cpu-baseline
b 7b_n16 --n 16 --no-cpu-baseline
b 13b_n8 --workload llama2-13b-decode --n 8 --no-cpu-baseline
b 70b_n8 --workload llama2-70b-decode --n 8 --no-cpu-baseline
