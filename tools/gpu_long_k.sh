#!/bin/bash
# Dispatch for long K at n >= 300: the persistent kernel only up to PERSIST_MAX_KT stages, and split-K 2 in
# several waves for 256-token tiles keeping >= 16 stages per CTA -- A/B on the (shape, n) these change.
set -u
O=gpurun_out/lk; mkdir -p $O; rm -f $O/t_*.jsonl
python -m paper_2311_02103_b200.build --experiments > $O/build.log 2>&1 || { echo BUILD_FAIL; exit 1; }
export RELAX_Q4_LIB=build_exp/librelax_q4_exp.so
SPECS=("11008x4096 1536" "13824x5120 1024,2048,3072,4096" "8192x8192 640,768,3072,4096" "8192x28672 640,768,1024,1536,2048,3072,4096" "28672x8192 640,768,2048,3072,4096" "8192x10240 512,1024,2048,3072,4096" "14336x4096 1536,4096" "8192x3584 1536,3072" "14336x8192 640,768,2048,3072,4096" "28672x4096 1536,4096")
for cfg in base new; do
  if [ $cfg = new ]; then export RELAX_Q4_PERSIST_MAX_KT=24 RELAX_Q4_MW_SPLIT_MIN_KS=16; fi
  for spec in "${SPECS[@]}"; do
    set -- $spec
    timeout 600 python tools/sweep.py --shapes $1 --ns $2 --variants auto --out $O/t_$cfg.jsonl > /dev/null 2>&1
  done
  echo "sweep $cfg done"
done
python - <<'PY'
import json
a={}
for c in ("base","new"):
    for l in open(f"gpurun_out/lk/t_{c}.jsonl"):
        d=json.loads(l)
        if 'us' in d: a.setdefault((d['K'],d['N'],d['n']),{})[c]=(d['us'],d['sched']['tile'],d['sched']['split_k'],d['sched'].get('persistent',False))
for k,x in sorted(a.items()):
    print(k, x.get("base"), x.get("new"), "x%.3f" % (x["base"][0]/x["new"][0]) if len(x)==2 else "")
PY
