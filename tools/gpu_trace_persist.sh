#!/bin/bash
# Stream-K timeline (experiments build, RELAX_Q4_TRACE=1) + parity + a short A/B sweep
set -u
O=gpurun_out/tp; mkdir -p $O
python -m paper_2311_02103_b200.build > $O/build.log 2>&1 || { echo BUILD_FAIL; exit 1; }
python -m paper_2311_02103_b200.build --experiments > $O/build_exp.log 2>&1 || { echo BUILD_FAIL; exit 1; }
timeout 600 python -m pytest tests/test_gpu_streamk.py -q -x --timeout 300 > $O/pytest_sk.log 2>&1; echo "pytest streamk rc=$?"; tail -2 $O/pytest_sk.log
for c in "4096 11008 512" "8192 28672 512" "4096 4096 2048" "4096 12288 512" "4096 22016 512"; do
  tag=$(echo $c | tr ' ' '_')
  RELAX_Q4_LIB=build_exp/librelax_q4_exp.so RELAX_Q4_TRACE=1 timeout 120 python tools/trace_persist.py $c --all > $O/tp_$tag.txt 2>&1; echo "trace $c rc=$? $(tail -1 $O/tp_$tag.txt)"
done
for sk in 0 1; do
  RELAX_Q4_LIB=build_exp/librelax_q4_exp.so RELAX_Q4_STREAMK=$sk timeout 900 python tools/sweep.py --shapes ${SHAPES:-4096x4096,4096x11008,4096x12288,4096x22016,4096x32000,8192x28672,11008x4096} \
      --ns ${NS:-300,512,777,1024,1536,2048} --variants auto --out $O/sweep_sk$sk.jsonl > /dev/null 2>&1; echo "sweep sk=$sk rc=$?"
done
python - <<'PY'
import json
a={}
for sk in (0,1):
    try:
        for l in open(f"gpurun_out/tp/sweep_sk{sk}.jsonl"):
            d=json.loads(l)
            if 'us' in d: a.setdefault((d['K'],d['N'],d['n']),{})[sk]=(d['us'],d['TFLOPS'],d['sched'].get('stream_k',False))
    except FileNotFoundError: pass
for k,v in sorted(a.items()):
    if 0 in v and 1 in v and v[1][2]: print(k, "sk0", v.get(0), "sk1", v.get(1), "x%.3f" % (v[0][0]/v[1][0]))
PY
