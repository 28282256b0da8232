#!/bin/bash
# A/B of the decode kernel's L2 prefetch of the rows beyond its ring (RELAX_Q4_GS_L2PF_KB, experiments build)
set -u
O=gpurun_out/l2pf; mkdir -p $O
python -m paper_2311_02103_b200.build --experiments > $O/build.log 2>&1 || { echo BUILD_FAIL; exit 1; }
export RELAX_Q4_LIB=build_exp/librelax_q4_exp.so
for wl in llama2-7b-decode llama2-13b-decode llama2-70b-decode; do
  for kb in 0 96 192 512 1024; do
    RELAX_Q4_GS_L2PF_KB=$kb timeout 300 python bench.py --workload $wl --no-cpu-baseline > $O/b_${wl}_$kb.json 2>/dev/null
    echo "$wl l2pf=${kb}KB $(python -c "import json; d=json.load(open('$O/b_${wl}_$kb.json')); print(d['value'], d['hbm_gbs'], d['roofline']['frac'], d['clocks']['reasons'])" 2>&1 | tail -1)"
  done
done
