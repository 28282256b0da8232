#!/bin/bash
# Stream-K vs the previous schedule choice (RELAX_Q4_STREAMK=0), experiments build, per shape and n
set -u
O=gpurun_out/sk; mkdir -p $O
python -m paper_2311_02103_b200.build --experiments > $O/build.log 2>&1 || { echo BUILD_FAIL; exit 1; }
export RELAX_Q4_LIB=build_exp/librelax_q4_exp.so
for sk in 0 1; do
  RELAX_Q4_STREAMK=$sk timeout 900 python tools/sweep.py --shapes 4096x4096,4096x11008,11008x4096,4096x12288,4096x22016,4096x32000 \
      --ns 256,512,1024,2048,4096 --variants auto --out $O/sweep_sk$sk.jsonl > /dev/null 2>&1
done
RELAX_Q4_STREAMK=1 timeout 600 python -m pytest tests/test_gpu_streamk.py -q 2>&1 | tail -2
python - <<'PY'
import json
a={}
for sk in (0,1):
    for l in open(f"gpurun_out/sk/sweep_sk{sk}.jsonl"):
        d=json.loads(l); a.setdefault((d['K'],d['N'],d['n']),{})[sk]=(d['us'],d['TFLOPS'],d['sched'].get('stream_k',False))
for k,v in sorted(a.items()):
    print(k, "sk0", v.get(0), "sk1", v.get(1))
PY
