#!/bin/bash
set -u
O=gpurun_out/grp; mkdir -p $O
python -m paper_2311_02103_b200.build > $O/build.log 2>&1 || { echo BUILD_FAIL; tail -5 $O/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_grouped.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -5 $O/pytest.log
b() { tag=$1; shift; timeout 900 python bench.py "$@" > $O/bench_$tag.json 2> $O/bench_$tag.err; echo "bench $tag rc=$? $(python -c "import json; d=json.load(open('$O/bench_$tag.json')); print(d['value'], d['hbm_gbs'], d['roofline']['frac'], d['gpu_launches'], d.get('serial_chain'), d['config']['workload'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>&1 | tail -1)"; tail -2 $O/bench_$tag.err; }
b 7b_decode
b 7b_serial --serial --no-cpu-baseline
b 13b --workload llama2-13b-decode --no-cpu-baseline
b 70b --workload llama2-70b-decode --no-cpu-baseline
b 7b_n2 --n 2 --no-cpu-baseline
b 7b_n8 --n 8 --no-cpu-baseline
