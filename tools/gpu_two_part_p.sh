#!/bin/bash
# Two-part schedule with the leading rows on the persistent kernel (RELAX_Q4_TWO_PART=1) vs without that
# variant (=2), experiments build; product parity of every schedule class.
set -u
O=gpurun_out/tp4; mkdir -p $O; rm -f $O/t_*.jsonl
python -m paper_2311_02103_b200.build > $O/build.log 2>&1 || { echo BUILD_FAIL; exit 1; }
python -m paper_2311_02103_b200.build --experiments > $O/build_exp.log 2>&1 || { echo BUILD_FAIL; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_schedules.py tests/test_gpu_parity.py tests/test_gpu_threads.py -q -x --timeout 600 > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
SPECS=("4096x11008 3584" "4096x32000 640,768" "4096x12288 2048,3584" "5120x32000 640,768,1536" "4096x14336 2048,3072" "4096x28672 1024,1536")
for v in 2 1; do
  for spec in "${SPECS[@]}"; do
    set -- $spec
    RELAX_Q4_LIB=build_exp/librelax_q4_exp.so RELAX_Q4_TWO_PART=$v timeout 600 python tools/sweep.py --shapes $1 --ns $2 --variants auto --out $O/t_$v.jsonl > /dev/null 2>&1
  done
done
python - <<'PY'
import json
a={}
for v in ("2","1"):
    for l in open(f"gpurun_out/tp4/t_{v}.jsonl"):
        d=json.loads(l)
        if 'us' in d: a.setdefault((d['K'],d['N'],d['n']),{})[v]=(d['us'],d['sched'])
for k,x in sorted(a.items()):
    if len(x)==2: print(k, "before %.1f" % x["2"][0], "persistent-A %.1f" % x["1"][0], "x%.3f" % (x["2"][0]/x["1"][0]))
PY
