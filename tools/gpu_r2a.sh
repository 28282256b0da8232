#!/bin/bash
set -u
O=gpurun_out/r2a; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo BUILD_FAIL; tail $O/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_tp.py tests/test_gpu_fused.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -5 $O/pytest.log
./tools/dispatch_cost > $O/dispatch_cost.txt 2>&1; echo "dispatch rc=$?"; cat $O/dispatch_cost.txt
b() { tag=$1; shift; timeout 900 python bench.py "$@" > $O/bench_$tag.json 2> $O/bench_$tag.err; echo "bench $tag rc=$? $(python -c "import json; d=json.load(open('$O/bench_$tag.json')); print(d['value'], d['roofline']['frac'], d['e2e']['value'], d.get('e2e_eager'), d['clocks'], d.get('cpu_baseline',{}).get('value'))" 2>&1 | tail -1)"; tail -3 $O/bench_$tag.err; }
b 7b_decode
b 7b_tp1 --tp --no-cpu-baseline
b 70b_tp1 --tp --workload llama2-70b-decode --no-cpu-baseline
b 7b_fused --fused --no-cpu-baseline
timeout 600 python bench.py --impl reference > $O/ref.json 2>&1; echo "ref rc=$?"; cut -c1-300 $O/ref.json
