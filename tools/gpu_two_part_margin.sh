#!/bin/bash
# Two-part schedule at a smaller model margin (RELAX_Q4_TWO_PART_MARGIN=0.97) vs off, experiments build;
# then the 7B / 13B prefill bench lines with the product build.
set -u
O=gpurun_out/tp3; mkdir -p $O; rm -f $O/t_*.jsonl
python -m paper_2311_02103_b200.build > $O/build.log 2>&1 || { echo BUILD_FAIL; exit 1; }
python -m paper_2311_02103_b200.build --experiments > $O/build_exp.log 2>&1 || { echo BUILD_FAIL; exit 1; }
SPECS=("4096x4096 1536" "4096x11008 512,1024,1536" "11008x4096 1536" "4096x32000 300,384,512" "4096x12288 512" "4096x22016 192,256,300,384,512,640,768" "5120x5120 1024,2048,3072" "5120x13824 300,384,512,640,768" "13824x5120 1024,2048,3072,4096" "8192x8192 640,768,2048,3072" "8192x28672 300,384,512,1024,1536,2048,3072" "28672x8192 640,768,2048,3072" "8192x10240 300,384,512,1024,1536,2048,3072" "14336x4096 1536" "4096x14336 640,768,1024" "8192x3584 1536,3072,4096" "3584x8192 640,768,2048" "14336x8192 640,768,2048,3072" "28672x4096 1536" "5120x32000 300,384,512" "8192x32000 300,384,512,640,768,1536")
for v in off m97; do
  for spec in "${SPECS[@]}"; do
    set -- $spec
    if [ $v = off ]; then
      RELAX_Q4_LIB=build_exp/librelax_q4_exp.so RELAX_Q4_TWO_PART=0 timeout 600 python tools/sweep.py --shapes $1 --ns $2 --variants auto --out $O/t_$v.jsonl > /dev/null 2>&1
    else
      RELAX_Q4_LIB=build_exp/librelax_q4_exp.so RELAX_Q4_TWO_PART_MARGIN=0.97 timeout 600 python tools/sweep.py --shapes $1 --ns $2 --variants auto --out $O/t_$v.jsonl > /dev/null 2>&1
    fi
  done
  echo "sweep $v done"
done
python - <<'PY'
import json
a={}
for v in ("off","m97"):
    for l in open(f"gpurun_out/tp3/t_{v}.jsonl"):
        d=json.loads(l)
        if 'us' in d: a.setdefault((d['K'],d['N'],d['n']),{})[v]=(d['us'],d['sched'].get('two_part',False))
for k,x in sorted(a.items()):
    if len(x)==2: print(k, "off %.1f" % x["off"][0], "m97 %.1f" % x["m97"][0], x["m97"][1], "x%.3f" % (x["off"][0]/x["m97"][0]))
PY
b() { tag=$1; shift; timeout 900 python bench.py "$@" > $O/bench_$tag.json 2> $O/bench_$tag.err; echo "bench $tag rc=$? $(python -c "import json; d=json.load(open('$O/bench_$tag.json')); print(d['value'], d['tflops'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>&1 | tail -1)"; }
b 7b_prefill_n512 --workload llama2-7b-prefill --n 512 --no-cpu-baseline
b 7b_prefill_n1024 --workload llama2-7b-prefill --n 1024 --no-cpu-baseline
b 13b_prefill_n512 --workload llama2-13b-prefill --n 512 --no-cpu-baseline
