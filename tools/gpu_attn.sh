#!/bin/bash
set -u
O=gpurun_out/attn; mkdir -p $O
python -m paper_2311_02103_b200.build > $O/build.log 2>&1 || { echo BUILD_FAIL; tail -5 $O/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_attention.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -15 $O/pytest.log
b() { tag=$1; shift; timeout 900 python bench.py "$@" > $O/bench_$tag.json 2> $O/bench_$tag.err; echo "bench $tag rc=$? $(python -c "import json; d=json.load(open('$O/bench_$tag.json')); print(d['value'], d['hbm_gbs'], d['roofline']['frac'], d['gpu_launches'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>&1 | tail -1)"; tail -2 $O/bench_$tag.err; }
b 7b_block_fused --block fused --no-cpu-baseline
b 7b_block_kv512 --block fused --kv 512 --no-cpu-baseline
b 7b_block_kv4096 --block fused --kv 4096 --no-cpu-baseline
b 70b_block_kv4096 --workload llama2-70b-decode --block fused --kv 4096 --no-cpu-baseline
