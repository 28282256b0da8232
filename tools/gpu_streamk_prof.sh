#!/bin/bash
# Stream-K diagnosis: parity, PDL on/off timing, ncu --set full of the stream-K and one-tile kernels at 4096 x 11008 n = 512
set -u
O=gpurun_out/skp; mkdir -p $O
python -m paper_2311_02103_b200.build > $O/build.log 2>&1 || { echo BUILD_FAIL; exit 1; }
timeout 900 python -m pytest tests/test_gpu_streamk.py tests/test_gpu_schedules.py -q -x --timeout 600 > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
for pd in "" "--no-pdl"; do
  timeout 300 python tools/sweep.py --shapes 4096x11008 --ns 512 --variants auto,tc-np $pd --out $O/sweep.jsonl 2>&1 | cut -c1-250
done
timeout 120 python tools/prof_one.py 4096 11008 512 auto 5 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:persist -s 2 -c 1 -o $O/prof_sk python tools/prof_one.py 4096 11008 512 auto 5 > $O/ncu_sk.log 2>&1; echo "ncu rc=$?"
ncu -i $O/prof_sk.ncu-rep --page details --csv > $O/prof_sk_details.csv 2>/dev/null
ncu -i $O/prof_sk.ncu-rep --page source --csv > $O/prof_sk_source.csv 2>/dev/null
ls -la $O
