#!/bin/bash
# Two-part TC schedule (whole 256-token tiles over the leading rows + a split-K launch for the rest rows):
# A/B RELAX_Q4_TWO_PART=0 vs 1 (experiments build) on every (shape, n) where the model offers it; product parity.
set -u
O=gpurun_out/tp2; mkdir -p $O; rm -f $O/t_*.jsonl
python -m paper_2311_02103_b200.build > $O/build.log 2>&1 || { echo BUILD_FAIL; exit 1; }
python -m paper_2311_02103_b200.build --experiments > $O/build_exp.log 2>&1 || { echo BUILD_FAIL; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_schedules.py tests/test_gpu_parity.py tests/test_gpu_threads.py -q -x --timeout 600 > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
SPECS=("4096x4096 1536" "4096x11008 512,1024" "4096x12288 512" "4096x22016 192,256,512" "5120x5120 1024,2048,3072" \
       "5120x13824 300,384,512,640,768" "13824x5120 1024,2048,3072" "8192x8192 640,768" "8192x28672 512,1024" \
       "28672x8192 640,768,2048,3072" "8192x10240 512,1024,1536" "4096x14336 768,1024" "8192x3584 1536,3072,4096" \
       "3584x8192 640,768" "14336x8192 640,768,2048" "2048x2000 3072")
export RELAX_Q4_LIB=build_exp/librelax_q4_exp.so
for v in 0 1; do
  for spec in "${SPECS[@]}"; do
    set -- $spec
    RELAX_Q4_TWO_PART=$v timeout 600 python tools/sweep.py --shapes $1 --ns $2 --variants auto --out $O/t_$v.jsonl > /dev/null 2>&1
  done
  echo "sweep $v done"
done
python - <<'PY'
import json
a={}
for v in ("0","1"):
    for l in open(f"gpurun_out/tp2/t_{v}.jsonl"):
        d=json.loads(l)
        if 'us' in d: a.setdefault((d['K'],d['N'],d['n']),{})[v]=(d['us'],d['sched'])
for k,x in sorted(a.items()):
    if len(x)==2: print(k, "off %.1f" % x["0"][0], "on %.1f" % x["1"][0], "x%.3f" % (x["0"][0]/x["1"][0]))
PY
