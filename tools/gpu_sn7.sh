#!/bin/bash
set -u
O=gpurun_out/sn7; mkdir -p $O
python -m paper_2311_02103_b200.build --experiments > $O/build.log 2>&1 || { echo BUILD_FAIL; tail -5 $O/build.log; exit 1; }
export RELAX_Q4_LIB=$PWD/build_exp/librelax_q4_exp.so
for cfg in "8192 1" "8192 1.5" "16384 1" "16384 2" "1073741824 2"; do
  set -- $cfg
  export RELAX_Q4_SMALLN_MAX_K=$1 RELAX_Q4_TC_CTAS_PER_SM=$2
  line="maxK=$1 tc_ctas=$2:"
  for spec in "7b:--n 8" "7bf:--fused --n 8" "13b:--workload llama2-13b-decode --n 8" "70b:--workload llama2-70b-decode --n 8" "70bf:--workload llama2-70b-decode --fused --n 8" "7b16:--n 16"; do
    tag=${spec%%:*}; fl=${spec#*:}
    v=$(timeout 600 python bench.py $fl --no-cpu-baseline 2>/dev/null | python -c "import json,sys; print(json.load(sys.stdin)['value'])")
    line="$line $tag=$v"
  done
  echo "$line"
done
