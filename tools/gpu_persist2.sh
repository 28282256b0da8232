#!/bin/bash
set -u
O=gpurun_out/persist2; mkdir -p $O
python -m paper_2311_02103_b200.build > $O/build.log 2>&1 || { echo BUILD_FAIL; tail -5 $O/build.log; exit 1; }
python -m paper_2311_02103_b200.build --experiments > $O/build_exp.log 2>&1 || { echo BUILD_FAIL; tail -5 $O/build_exp.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "tc256p or prefix or llama_shapes or random" > $O/pytest1.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest1.log
export RELAX_Q4_LIB=$PWD/build_exp/librelax_q4_exp.so RELAX_Q4_PERSIST_MIN_TILES=0
timeout 1500 python tools/sweep.py --shapes 4096x4096,4096x11008,11008x4096,4096x32000 --ns 256,512,1024,2048,4096 --variants auto,auto-np --out $O/sweep.jsonl > $O/sweep.log 2>&1; echo "sweep rc=$?"
python -c "
import json
rows=[json.loads(l) for l in open('$O/sweep.jsonl')]
d={}
for r in rows:
    if 'us' in r: d.setdefault((r['K'],r['N'],r['n']),{})[r['variant']]=(r['us'],r['TFLOPS'])
for k in sorted(d): print(k, d[k])
"
unset RELAX_Q4_LIB RELAX_Q4_PERSIST_MIN_TILES
for nn in 512 4096; do timeout 600 python bench.py --workload llama2-7b-prefill --n $nn --steps 5 --no-cpu-baseline > $O/bench_$nn.json 2>$O/bench_$nn.err; echo "bench n=$nn: $(python -c "import json; d=json.load(open('$O/bench_$nn.json')); print(d['value'], d['tflops'], d['roofline']['frac'], d['clocks'])" 2>&1|tail -1)"; done
