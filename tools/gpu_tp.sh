#!/bin/bash
set -u
O=gpurun_out/tp; mkdir -p $O
python -m paper_2311_02103_b200.build > $O/build.log 2>&1 || { echo BUILD_FAIL; tail -5 $O/build.log; exit 1; }
b() { tag=$1; shift; timeout 900 python bench.py "$@" > $O/bench_$tag.json 2> $O/bench_$tag.err; echo "bench $tag rc=$? $(python -c "import json; d=json.load(open('$O/bench_$tag.json')); print(d['value'], d['hbm_gbs'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>&1 | tail -1)"; }
for p in 1 2 4 8; do
  b 70b_fused_shard$p --workload llama2-70b-decode --fused --tp-shard $p --no-cpu-baseline
  b 70b_shard$p --workload llama2-70b-decode --tp-shard $p --no-cpu-baseline
done
b 70b_megatron_tp1 --workload llama2-70b-decode --tp --no-cpu-baseline
b 7b_megatron_tp1 --tp --no-cpu-baseline
