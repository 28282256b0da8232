#!/bin/bash
# F1: Megatron TP decode at NCCL world 1 with the row-split sums fused into the
# decode kernel (default) vs an NCCL all_reduce (--nccl-allreduce)
set -u
O=gpurun_out/tp_ar; mkdir -p $O
python -m paper_2311_02103_b200.build > $O/build.log 2>&1 || { echo BUILD_FAIL; tail -5 $O/build.log; exit 1; }
b() { tag=$1; shift; timeout 900 python bench.py "$@" > $O/bench_$tag.json 2> $O/bench_$tag.err; echo "bench $tag rc=$? $(python -c "import json; d=json.load(open('$O/bench_$tag.json')); print(d['value'], d['hbm_gbs'], d['roofline']['frac'], d['config'].get('tp_allreduce'), d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>&1 | tail -1)"; }
b 7b_tp1_fusedar --tp --no-cpu-baseline
b 7b_tp1_nccl --tp --nccl-allreduce --no-cpu-baseline
b 70b_tp1_fusedar --workload llama2-70b-decode --tp --no-cpu-baseline
b 70b_tp1_nccl --workload llama2-70b-decode --tp --nccl-allreduce --no-cpu-baseline
b 7b_fused_plain --fused --no-cpu-baseline
