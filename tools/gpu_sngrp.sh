#!/bin/bash
set -u
O=gpurun_out/sngrp; mkdir -p $O
python -m paper_2311_02103_b200.build > $O/build.log 2>&1 || { echo BUILD_FAIL; tail -5 $O/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_grouped.py -x -q 2>&1 | tail -3
b() { tag=$1; shift; timeout 900 python bench.py "$@" > $O/bench_$tag.json 2> $O/bench_$tag.err; echo "bench $tag rc=$? $(python -c "import json; d=json.load(open('$O/bench_$tag.json')); print(d['value'], d['hbm_gbs'], d['roofline']['frac'], d['gpu_launches'], (d.get('serial_chain') or {}).get('value'), d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>&1 | tail -1)"; }
for n in 3 4 8; do b 7b_n$n --n $n --no-cpu-baseline; done
b 13b_n8 --workload llama2-13b-decode --n 8 --no-cpu-baseline
b 70b_n8 --workload llama2-70b-decode --n 8 --no-cpu-baseline
