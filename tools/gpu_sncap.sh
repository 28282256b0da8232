#!/bin/bash
# small-batch kernel: shared-memory cap (ring depth) A/B, experiments build
set -u
python -m paper_2311_02103_b200.build --experiments > /dev/null 2>&1 || { echo BUILD_FAIL; exit 1; }
export RELAX_Q4_LIB=build_exp/librelax_q4_exp.so
for kb in 113 160 220; do
  echo "== cap ${kb} KB"
  RELAX_Q4_SN_SMEM_KB=$kb timeout 120 python tools/trace_smalln.py --layers 3 --n 8 2>&1 | tail -5
  for n in 4 8; do
    RELAX_Q4_SN_SMEM_KB=$kb timeout 300 python bench.py --n $n --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('cap $kb n=$n', d['value'], d['hbm_gbs'], d['roofline']['frac'])"
  done
done
