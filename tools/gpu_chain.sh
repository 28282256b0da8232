#!/bin/bash
set -u
O=gpurun_out/chain; mkdir -p $O
# the decode chain lives in the experiments build (include/relax_q4_debug.h)
python -m paper_2311_02103_b200.build > $O/build.log 2>&1 || { echo BUILD_FAIL; tail -5 $O/build.log; exit 1; }
python -m paper_2311_02103_b200.build --experiments >> $O/build.log 2>&1 || { echo BUILD_FAIL; exit 1; }
export RELAX_Q4_LIB=build_exp/librelax_q4_exp.so
CUDA_VISIBLE_DEVICES="" python tests/_abi_fake_ptr.py | tail -2
timeout 300 python -m pytest tests/test_gpu_chain.py -x -q 2>&1 | tail -15
b() { tag=$1; shift; timeout 600 python bench.py "$@" > $O/bench_$tag.json 2> $O/bench_$tag.err; echo "bench $tag rc=$? $(python -c "import json; d=json.load(open('$O/bench_$tag.json')); print(d['value'], d['hbm_gbs'], d['roofline']['frac'], d['gpu_launches'], (d.get('serial_chain') or {}).get('value'), d['e2e']['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>&1 | tail -1)"; }
b 7b_chain --chain --no-cpu-baseline
b 7b_default --no-cpu-baseline
b 13b_chain --workload llama2-13b-decode --chain --no-cpu-baseline
b 70b_chain --workload llama2-70b-decode --chain --no-cpu-baseline
b 7b_chain_fused --chain --fused --no-cpu-baseline
