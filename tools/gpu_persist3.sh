#!/bin/bash
set -u
O=gpurun_out/persist3; mkdir -p $O
python -m paper_2311_02103_b200.build > $O/build.log 2>&1 || { echo BUILD_FAIL; tail -5 $O/build.log; exit 1; }
python -m paper_2311_02103_b200.build --experiments > $O/build_exp.log 2>&1 || { echo BUILD_FAIL; tail -5 $O/build_exp.log; exit 1; }
export RELAX_Q4_LIB=$PWD/build_exp/librelax_q4_exp.so
RELAX_Q4_PERSIST_BN=128 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "prefix or llama_shapes" > $O/pytest128.log 2>&1; echo "pytest persist128 rc=$?"; tail -2 $O/pytest128.log
for cfg in "p128:RELAX_Q4_PERSIST_BN=128" "p256:RELAX_Q4_PERSIST_BN=256" "np:RELAX_Q4_PERSIST=0"; do
  tag=${cfg%%:*}; kv=${cfg#*:}
  env $kv timeout 1500 python tools/sweep.py --shapes 4096x4096,4096x11008,11008x4096,4096x32000 --ns 256,512,1024,4096 --variants auto --out $O/sweep_$tag.jsonl > /dev/null 2>&1
done
python - <<'PY'
import json
d={}
for tag in ("p128","p256","np"):
    for l in open(f"gpurun_out/persist3/sweep_{tag}.jsonl"):
        r=json.loads(l)
        if 'us' in r: d.setdefault((r['K'],r['N'],r['n']),{})[tag]=r['TFLOPS']
for k in sorted(d): print(k, d[k])
PY
