#!/bin/bash
set -u
O=gpurun_out/sn4; mkdir -p $O
python -m paper_2311_02103_b200.build > /dev/null 2>&1; python -m paper_2311_02103_b200.build --experiments > /dev/null 2>&1
export RELAX_Q4_LIB=$PWD/build_exp/librelax_q4_exp.so
for cfg in "8 1" "16 1" "8 2" "16 2"; do
  set -- $cfg
  export RELAX_Q4_SN_WARPS=$1 RELAX_Q4_SN_GRID_MULT=$2
  timeout 1200 python tools/sweep.py --shapes 4096x4096,4096x11008,11008x4096,4096x32000,8192x8192,28672x8192 --ns 2,8 --variants smalln --out $O/sweep_w$1_g$2.jsonl > /dev/null 2>&1
  b=$(timeout 600 python bench.py --n 8 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['value'], d['hbm_gbs'])")
  b2=$(timeout 600 python bench.py --n 2 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['value'], d['hbm_gbs'])")
  echo "W=$1 mult=$2 bench n=8: $b  n=2: $b2"
  python -c "
import json
for l in open('$O/sweep_w$1_g$2.jsonl'):
    r=json.loads(l)
    if 'us' in r: print('   ', r['K'],r['N'],r['n'],r['us'],r['GBps'])
"
done
