#!/bin/bash
# Dispatch model: cost of an unamortised split-K cluster reduction (<= 2 stages per CTA):
# RELAX_Q4_SPLIT_SHORT_US 1.0 (old model) vs 3.0, on the (shape, n) whose choice it changes
set -u
O=gpurun_out/spl; mkdir -p $O; rm -f $O/t_*.jsonl
python -m paper_2311_02103_b200.build --experiments > $O/build.log 2>&1 || { echo BUILD_FAIL; exit 1; }
export RELAX_Q4_LIB=build_exp/librelax_q4_exp.so
for v in 1.0 3.0; do
  for spec in "1024x1024 65,256,1024" "1024x2048 128,512" "1024x4096 65,256" "1024x8192 65,128" "2048x1024 65,256,512" \
              "2048x4096 96" "3584x1024 128" "4096x1024 65,128" "2048x2048 128,256"; do
    set -- $spec
    RELAX_Q4_SPLIT_SHORT_US=$v timeout 300 python tools/sweep.py --shapes $1 --ns $2 --variants auto --out $O/t_$v.jsonl > /dev/null 2>&1
  done
  echo "sweep $v done"
done
python - <<'PY'
import json
a={}
for v in ("1.0","3.0"):
    for l in open(f"gpurun_out/spl/t_{v}.jsonl"):
        d=json.loads(l)
        if 'us' in d: a.setdefault((d['K'],d['N'],d['n']),{})[v]=(d['us'],d['sched']['tile'],d['sched']['split_k'])
for k,x in sorted(a.items()):
    print(k, x.get("1.0"), x.get("3.0"), "x%.3f" % (x["1.0"][0]/x["3.0"][0]) if len(x)==2 else "")
PY
