#!/bin/bash
O=gpurun_out/prof_persist; mkdir -p $O
python -m paper_2311_02103_b200.build > $O/build.log 2>&1 || { echo BUILD_FAIL; exit 1; }
timeout 120 python tools/prof_one.py 4096 11008 4096 auto 3 > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:persist -s 1 -c 1 -o $O/persist_4096x11008_n4096 python tools/prof_one.py 4096 11008 4096 auto 3 > $O/ncu.log 2>&1
echo "ncu rc=$?"
bash tools/ncu_summary.sh $O/persist_4096x11008_n4096.ncu-rep
ncu -i $O/persist_4096x11008_n4096.ncu-rep --page details --csv 2>/dev/null | grep -i "shared\|L2 Cache Throughput\|L1/TEX Cache Throughput\|Memory Throughput\|Compute (SM)" | head -20
