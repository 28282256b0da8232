#!/bin/bash
# Pair-MMA (tcgen05 cta_group::2) form of the persistent kernel: parity under trapping waits (debug
# experiments build, every n > 64 TC call forced persistent), then timing C2=0 vs 1 (experiments build).
set -u
O=gpurun_out/c2; mkdir -p $O
RELAX_Q4_DEBUG=1 python -m paper_2311_02103_b200.build --experiments > $O/build_dbg.log 2>&1 || { echo BUILD_FAIL; tail -5 $O/build_dbg.log; exit 1; }
export RELAX_Q4_LIB=build_exp/librelax_q4_exp.so
RELAX_Q4_PERSIST_C2=1 RELAX_Q4_PERSIST_BN=256 timeout 300 python tools/prof_one.py 4096 4096 512 tc 2 > $O/one.log 2>&1; echo "one call rc=$?"; tail -3 $O/one.log
RELAX_Q4_PERSIST_C2=1 RELAX_Q4_PERSIST_BN=256 timeout 900 python -m pytest tests/test_gpu_schedules.py tests/test_gpu_parity.py -q -x --timeout 300 > $O/pytest_c2_dbg.log 2>&1; echo "pytest c2 (debug) rc=$?"; tail -3 $O/pytest_c2_dbg.log
python -m paper_2311_02103_b200.build --experiments > $O/build.log 2>&1 || { echo BUILD_FAIL; exit 1; }
for c2 in 0 1; do
  RELAX_Q4_PERSIST_C2=$c2 RELAX_Q4_PERSIST_BN=256 timeout 900 python tools/sweep.py --shapes ${SHAPES:-4096x4096,4096x11008,11008x4096,4096x32000,8192x28672} \
     --ns ${NS:-512,1024,2048,4096} --variants auto --out $O/sweep_c2_$c2.jsonl > /dev/null 2>&1; echo "sweep c2=$c2 rc=$?"
done
python - <<'PY'
import json
a={}
for c in (0,1):
    try:
        for l in open(f"gpurun_out/c2/sweep_c2_{c}.jsonl"):
            d=json.loads(l)
            if 'us' in d: a.setdefault((d['K'],d['N'],d['n']),{})[c]=(d['us'],d['TFLOPS'])
    except FileNotFoundError: pass
for k,v in sorted(a.items()):
    print(k, "c2=0", v.get(0), "c2=1", v.get(1), "x%.3f" % (v[0][0]/v[1][0]) if 0 in v and 1 in v else "")
PY
