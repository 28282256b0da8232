#!/bin/bash
# Config sweeps: c3 7B prefill n-sweep, c4 13B, c5 70B + TP shards.
set -u
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD_FAIL; exit 1; }
NS_C3="1,2,3,4,5,6,7,8,9,10,11,12,13,14,15,16,17,24,32,48,64,80,96,100,128,192,256,384,512,768,1000,1024,1536,2048,3072,4095,4096"
timeout 1200 python tools/sweep.py --shapes 4096x4096,4096x11008,11008x4096,4096x32000 --ns $NS_C3 --variants auto --reps 5 --out gpurun_out/sweep_c3.jsonl > gpurun_out/sweep_c3.log 2>&1; echo "c3 rc=$?"
timeout 600 python tools/sweep.py --shapes 4096x4096,4096x11008,11008x4096,4096x32000 --ns 1,2,3,4,5,6,8,12,16 --variants gemv,tc --reps 5 --out gpurun_out/sweep_cross.jsonl > gpurun_out/sweep_cross.log 2>&1; echo "cross rc=$?"
timeout 900 python tools/sweep.py --shapes 5120x5120,5120x13824,13824x5120,5120x32000 --ns 1,2,4,8,16,32,64,128,256,512,1024,2048,4096 --variants auto --reps 5 --out gpurun_out/sweep_c4.jsonl > gpurun_out/sweep_c4.log 2>&1; echo "c4 rc=$?"
timeout 1200 python tools/sweep.py --shapes 8192x8192,8192x1024,8192x28672,28672x8192,8192x32000,8192x4096,4096x8192,8192x512,8192x14336,14336x8192,8192x2048,2048x8192,8192x7168,7168x8192,8192x3584,3584x8192,8192x256,8192x128 --ns 1,16,128,512,4096 --variants auto --reps 3 --out gpurun_out/sweep_c5.jsonl > gpurun_out/sweep_c5.log 2>&1; echo "c5 rc=$?"
