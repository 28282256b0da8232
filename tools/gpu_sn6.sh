#!/bin/bash
set -u
O=gpurun_out/sn6; mkdir -p $O
python -m paper_2311_02103_b200.build --experiments > $O/build.log 2>&1 || { echo BUILD_FAIL; tail -5 $O/build.log; exit 1; }
export RELAX_Q4_LIB=$PWD/build_exp/librelax_q4_exp.so
for rep in 1 2; do
for mk in 5120 8192 1073741824; do
  export RELAX_Q4_SMALLN_MAX_K=$mk
  line="maxK=$mk rep=$rep:"
  for spec in "7b:--n 8" "7bf:--fused --n 8" "13b:--workload llama2-13b-decode --n 8" "70b:--workload llama2-70b-decode --n 8" "7b4:--n 4"; do
    tag=${spec%%:*}; fl=${spec#*:}
    v=$(timeout 600 python bench.py $fl --no-cpu-baseline 2>/dev/null | python -c "import json,sys; print(json.load(sys.stdin)['value'])")
    line="$line $tag=$v"
  done
  echo "$line"
done
done
