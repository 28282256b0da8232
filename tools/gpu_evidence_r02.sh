#!/bin/bash
# Round-2 evidence pass on one GPU: build, smoke, pytest -m gpu, bench lines,
# the oracle reference arm, ncu launch lists of the decode steps and ncu
# --set full of the decode GEMV, the small-n kernel and the tensor-core kernels.
set -u
O=gpurun_out/ev2; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo BUILD_FAIL; tail $O/build.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
if [ "${SKIP_TESTS:-0}" != "1" ]; then
  timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
fi
b() { tag=$1; shift; timeout 900 python bench.py "$@" > $O/bench_$tag.json 2> $O/bench_$tag.err; echo "bench $tag rc=$? $(python -c "import json; d=json.load(open('$O/bench_$tag.json')); print(d['value'], d['hbm_gbs'], d['tflops'], d['roofline']['frac'], d['e2e']['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>&1 | tail -1)"; }
b 7b_decode
b 7b_decode_fused --fused --no-cpu-baseline
b 13b_decode --workload llama2-13b-decode --no-cpu-baseline
b 13b_decode_fused --workload llama2-13b-decode --fused --no-cpu-baseline
b 70b_decode --workload llama2-70b-decode --no-cpu-baseline
b 70b_decode_fused --workload llama2-70b-decode --fused --no-cpu-baseline
for nn in 2 4 8 16 32; do b 7b_decode_batch$nn --n $nn --no-cpu-baseline; done
b 7b_decode_fused_batch8 --fused --n 8 --no-cpu-baseline
b 13b_decode_batch8 --workload llama2-13b-decode --n 8 --no-cpu-baseline
b 7b_block_fused --block fused --no-cpu-baseline
b 7b_block_unfused --block unfused --no-cpu-baseline
b 7b_block_fused_kv512 --block fused --kv 512 --no-cpu-baseline
b 7b_block_fused_kv4096 --block fused --kv 4096 --no-cpu-baseline
b 70b_block_fused_kv4096 --workload llama2-70b-decode --block fused --kv 4096 --no-cpu-baseline
b 7b_prefill_n128 --workload llama2-7b-prefill --n 128 --no-cpu-baseline
b 7b_prefill_n512 --workload llama2-7b-prefill --n 512 --no-cpu-baseline
b 7b_prefill_n4096 --workload llama2-7b-prefill --n 4096 --steps 5 --no-cpu-baseline
b 13b_prefill_n512 --workload llama2-13b-prefill --n 512 --no-cpu-baseline
b 7b_decode_serial --serial --no-cpu-baseline
b 70b_megatron_tp1 --workload llama2-70b-decode --tp --no-cpu-baseline
b 70b_megatron_tp1_nccl --workload llama2-70b-decode --tp --nccl-allreduce --no-cpu-baseline
b 7b_megatron_tp1 --tp --no-cpu-baseline
b 7b_megatron_tp1_nccl --tp --nccl-allreduce --no-cpu-baseline
for p in 2 4 8; do b 70b_fused_shard$p --workload llama2-70b-decode --fused --tp-shard $p --no-cpu-baseline; done
timeout 600 python bench.py --impl reference > $O/reference.json 2> $O/reference.err; echo "reference rc=$? $(cut -c1-200 $O/reference.json)"
if [ "${NCU:-1}" = "1" ]; then
  for spec in "7b:llama2-7b-decode-grouped-qkv-gateup:n1:" "7bfused:llama2-7b-decode-fused-qkv-gateup:n1:--fused" \
              "7bn8:llama2-7b-decode-grouped-qkv-gateup:n8:--n 8" "7bserial:llama2-7b-decode:n1:--serial"; do
    tag=${spec%%:*}; rest=${spec#*:}; key=${rest%:*}; fl=${rest##*:}
    timeout 600 python bench.py $fl --steps 2 --warmup 3 --no-cpu-baseline > $O/ll_plain_$tag.log 2>&1 && \
    timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 400 -c 300 --csv \
        --log-file $O/launches_$tag.csv python bench.py $fl --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_ll_$tag.log 2>&1
    echo "launch list $tag rc=$?"
    python tools/launch_summary.py $O/launches_$tag.csv $O/launches_${tag}_summary.csv "$key" > $O/launches_${tag}_shares.txt 2>&1
  done
  p() { tag=$1; kre=$2; shift 2; timeout 120 python tools/prof_one.py "$@" 5 > /dev/null 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kre -s 2 -c 1 -o $O/prof_$tag python tools/prof_one.py "$@" 5 > $O/ncu_$tag.log 2>&1; echo "ncu $tag rc=$?"; }
  p decode_4096x11008_n1 decode_stream 4096 11008 1 auto
  p decode_4096x4096_n1 decode_stream 4096 4096 1 auto
  p smalln_4096x11008_n8 smalln 4096 11008 8 auto
  p tc_4096x11008_n512 tc_q4 4096 11008 512 auto
  p persist_4096x32000_n4096 persist 4096 32000 4096 auto
  timeout 60 python tools/prof_attn.py 1 32 32 4096 3 > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_partial -s 2 -c 1 -o $O/prof_attn_b1_h32_L4096 python tools/prof_attn.py 1 32 32 4096 3 > $O/ncu_attn.log 2>&1; echo "ncu attn rc=$?"
fi
