#!/bin/bash
set -u
O=gpurun_out/idp; mkdir -p $O
python -m paper_2311_02103_b200.build > $O/build.log 2>&1 || { echo BUILD_FAIL; tail -5 $O/build.log; exit 1; }
./tools/ubench_idp > $O/ubench_idp.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -5 $O/pytest.log
b() { tag=$1; shift; timeout 900 python bench.py "$@" > $O/bench_$tag.json 2> $O/bench_$tag.err; echo "bench $tag rc=$? $(python -c "import json; d=json.load(open('$O/bench_$tag.json')); print(d['value'], d['hbm_gbs'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>&1 | tail -1)"; }
b 7b_decode --no-cpu-baseline
b 7b_fused --fused --no-cpu-baseline
b 13b --workload llama2-13b-decode --no-cpu-baseline
b 70b --workload llama2-70b-decode --no-cpu-baseline
b 7b_n2 --n 2 --no-cpu-baseline
b 7b_block --block fused --no-cpu-baseline
timeout 600 python tools/sweep.py --shapes 4096x4096,4096x11008,11008x4096,4096x32000 --ns 1,2 --variants auto --out $O/sweep.jsonl > /dev/null 2>&1
python -c "
import json
for l in open('$O/sweep.jsonl'):
    r=json.loads(l)
    if 'us' in r: print(r['K'],r['N'],r['n'],r['us'],r['GBps'])
"
