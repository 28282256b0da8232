#!/bin/bash
# Product build after the long-K dispatch change: parity of every schedule class, and timing on the changed points
set -u
O=gpurun_out/lkv; mkdir -p $O; rm -f $O/t.jsonl
python -m paper_2311_02103_b200.build > $O/build.log 2>&1 || { echo BUILD_FAIL; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_schedules.py tests/test_gpu_parity.py tests/test_gpu_threads.py -q --timeout 600 > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
for spec in "11008x4096 1536" "13824x5120 1024,4096" "8192x8192 640,768,3072,4096" "8192x28672 640,1024,2048,4096" "28672x8192 640,768,3072,4096" "8192x10240 512,2048,4096" "14336x4096 1536" "8192x3584 1536" "14336x8192 640,768,3072,4096" "28672x4096 1536"; do
  set -- $spec
  timeout 600 python tools/sweep.py --shapes $1 --ns $2 --variants auto --out $O/t.jsonl > /dev/null 2>&1
done
echo sweep done
