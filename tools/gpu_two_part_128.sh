#!/bin/bash
# Two-part schedule with 128-token tiles (RELAX_Q4_TWO_PART_BN128=1 vs 0), experiments build, on the points it changes;
# product parity of every schedule class.
set -u
O=gpurun_out/tp5; mkdir -p $O; rm -f $O/t_*.jsonl
python -m paper_2311_02103_b200.build > $O/build.log 2>&1 || { echo BUILD_FAIL; exit 1; }
python -m paper_2311_02103_b200.build --experiments > $O/build_exp.log 2>&1 || { echo BUILD_FAIL; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_schedules.py tests/test_gpu_parity.py -q -x --timeout 600 > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
SPECS=("11008x4096 640" "4096x22016 65,96,128" "13824x5120 512" "8192x10240 160,192,256" "8192x57344 65,96,128" "4096x14336 300,384")
for v in 0 1; do
  for spec in "${SPECS[@]}"; do
    set -- $spec
    RELAX_Q4_LIB=build_exp/librelax_q4_exp.so RELAX_Q4_TWO_PART_BN128=$v timeout 600 python tools/sweep.py --shapes $1 --ns $2 --variants auto --out $O/t_$v.jsonl > /dev/null 2>&1
  done
done
python - <<'PY'
import json
a={}
for v in ("0","1"):
    for l in open(f"gpurun_out/tp5/t_{v}.jsonl"):
        d=json.loads(l)
        if 'us' in d: a.setdefault((d['K'],d['N'],d['n']),{})[v]=(d['us'],d['TFLOPS'])
for k,x in sorted(a.items()):
    if len(x)==2: print(k, "before %.1f" % x["0"][0], "bn128 two-part %.1f" % x["1"][0], "x%.3f" % (x["0"][0]/x["1"][0]))
PY
