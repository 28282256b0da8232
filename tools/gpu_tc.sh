#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD_FAIL; exit 1; }
for f in 1 2; do
  RELAX_Q4_TC_CTAS_PER_SM=$f timeout 600 python tools/sweep.py --shapes 4096x4096,4096x11008,11008x4096,4096x32000 --ns 1,16,64 --variants tc,gemv --reps 5 --out gpurun_out/sweep_tc_f$f.jsonl > /dev/null 2>&1
  echo "f=$f"; python - <<PY
import json
for l in open("gpurun_out/sweep_tc_f$f.jsonl"):
    r=json.loads(l)
    if 'error' in r: print(r); continue
    print(f"{r['K']:>6}x{r['N']:<6} n={r['n']:<4} {r['variant']:<5} {r['us']:>8.2f}us {r['GBps']:>7.0f}GB/s sched={r['sched']['variant']}/{r['sched']['tile']}/s{r['sched']['split_k']}")
PY
done
timeout 100 python tools/prof_one.py 4096 11008 1 tc 5 > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_q4 -s 2 -c 1 -o gpurun_out/prof_tc_n1 python tools/prof_one.py 4096 11008 1 tc 5 > gpurun_out/ncu_tc.log 2>&1; echo ncu rc=$?
