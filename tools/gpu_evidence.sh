#!/bin/bash
# Evidence pass on one GPU: smoke, GPU tests, bench lines (7B decode default +
# fused, 13B, 70B, prefill), oracle reference arm, launch lists of the decode
# steps, ncu --set full of the dominant decode kernel and the TC GEMM.
set -u
mkdir -p gpurun_out/ev
O=gpurun_out/ev
timeout 300 python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo BUILD_FAIL; exit 1; }
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
if [ "${SKIP_TESTS:-0}" != "1" ]; then
  timeout 1500 python -m pytest tests -m gpu -q --timeout 600 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
fi
b() { tag=$1; shift; timeout 900 python bench.py "$@" > $O/bench_$tag.json 2> $O/bench_$tag.err; echo "bench $tag rc=$? $(cut -c1-160 $O/bench_$tag.json)"; }
b 7b_decode
b 7b_decode_fused --fused --no-cpu-baseline
b 13b_decode --workload llama2-13b-decode --no-cpu-baseline
b 13b_decode_fused --workload llama2-13b-decode --fused --no-cpu-baseline
b 7b_decode_batch2 --n 2 --no-cpu-baseline
b 7b_decode_batch8 --n 8 --no-cpu-baseline
b 7b_decode_batch32 --n 32 --no-cpu-baseline
b 7b_decode_fused_batch8 --fused --n 8 --no-cpu-baseline
b 7b_decode_fused_batch32 --fused --n 32 --no-cpu-baseline
b 7b_block_fused --block fused --no-cpu-baseline
b 7b_block_unfused --block unfused --no-cpu-baseline
b 13b_block_fused --workload llama2-13b-decode --block fused --no-cpu-baseline
b 13b_block_unfused --workload llama2-13b-decode --block unfused --no-cpu-baseline
b 70b_decode --workload llama2-70b-decode --no-cpu-baseline
b 70b_decode_fused --workload llama2-70b-decode --fused --no-cpu-baseline
b 7b_prefill_n512 --workload llama2-7b-prefill --n 512 --no-cpu-baseline
b 7b_prefill_n128 --workload llama2-7b-prefill --n 128 --no-cpu-baseline
b 7b_prefill_n4096 --workload llama2-7b-prefill --n 4096 --steps 5 --no-cpu-baseline
for p in 2 4 8; do b 70b_tp${p}_shard --workload llama2-70b-decode --tp-shard $p --no-cpu-baseline; done
b 70b_tp8_shard_fused --workload llama2-70b-decode --tp-shard 8 --fused --no-cpu-baseline
b reference --impl reference --steps 2
if [ "${NCU:-1}" = "1" ]; then
  for spec in "7b:" "7bfused:--fused"; do
    tag=${spec%%:*}; fl=${spec#*:}
    timeout 600 python bench.py $fl --steps 2 --warmup 3 --no-cpu-baseline > $O/ll_plain_$tag.log 2>&1 && \
    timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 800 -c 300 --csv \
        --log-file $O/launches_$tag.csv python bench.py $fl --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_ll_$tag.log 2>&1
    echo "launch list $tag rc=$?"
  done
  timeout 100 python tools/prof_one.py 4096 11008 1 auto 5 > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv -s 2 -c 1 -o $O/prof_gemv_4096x11008_n1 python tools/prof_one.py 4096 11008 1 auto 5 > $O/ncu1.log 2>&1; echo "ncu gemv rc=$?"
  timeout 100 python tools/prof_one.py 4096 11008 512 auto 5 > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_q4 -s 2 -c 1 -o $O/prof_tc_4096x11008_n512 python tools/prof_one.py 4096 11008 512 auto 5 > $O/ncu2.log 2>&1; echo "ncu tc rc=$?"
fi
