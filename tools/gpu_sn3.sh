#!/bin/bash
set -u
O=gpurun_out/sn3; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo BUILD_FAIL; tail $O/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "smalln" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
timeout 1200 python tools/sweep.py --shapes 4096x4096,4096x11008,11008x4096,4096x32000,5120x13824,13824x5120,8192x8192,28672x8192,8192x1024 --ns 2,8 --variants smalln --out $O/sweep_sn.jsonl > $O/sweep.log 2>&1; echo "sweep rc=$?"
timeout 120 python tools/prof_one.py 4096 32000 8 smalln 5 > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:smalln -s 2 -c 1 -o $O/sn_4096x32000_n8 python tools/prof_one.py 4096 32000 8 smalln 5 > $O/ncu.log 2>&1; bash tools/ncu_summary.sh $O/sn_4096x32000_n8.ncu-rep
