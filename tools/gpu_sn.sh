#!/bin/bash
set -u
O=gpurun_out/sn; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo BUILD_FAIL; tail $O/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "smalln or zero or config1 or random or bench_configuration or prefix" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -5 $O/pytest.log
timeout 900 python tools/sweep.py --shapes 4096x4096,4096x11008,11008x4096,4096x32000 --ns 1,2,3,4,6,8,12,16,24,32 --variants smalln,tc,auto --out $O/sweep_sn.jsonl > $O/sweep.log 2>&1; echo "sweep rc=$?"
python tools/summarize_sweep.py $O/sweep_sn.jsonl 2>&1 | head -60
for nn in 2 4 8 16; do timeout 600 python bench.py --n $nn --no-cpu-baseline > $O/bench_n$nn.json 2>$O/bench_n$nn.err; echo "bench n=$nn: $(python -c "import json; d=json.load(open('$O/bench_n$nn.json')); print(d['value'], d['hbm_gbs'], d['roofline']['frac'])" 2>&1|tail -1)"; done
