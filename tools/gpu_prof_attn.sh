#!/bin/bash
O=gpurun_out/prof_attn; mkdir -p $O
python -m paper_2311_02103_b200.build > $O/build.log 2>&1 || { echo BUILD_FAIL; exit 1; }
python tools/prof_attn.py 1 32 32 4096
python tools/prof_attn.py 1 64 8 4096
python tools/prof_attn.py 8 32 32 4096
timeout 600 ncu --set full --clock-control none -k regex:attn_partial -s 2 -c 1 -o $O/attn_7b python tools/prof_attn.py 1 32 32 4096 3 > $O/ncu.log 2>&1; echo "ncu rc=$?"
bash tools/ncu_summary.sh $O/attn_7b.ncu-rep
