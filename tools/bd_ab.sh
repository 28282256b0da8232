#!/bin/bash
# Block-diagonal warp-MMA decode GEMV (RELAX_Q4_GEMV_IMPL=bdmma) vs the streamed default.
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_gemv_impls.py -x -q 2>&1 | tail -3
val() { python -c "import json;d=json.load(open('$1'));print(d['value'])"; }
for v in "X=1" "RELAX_Q4_GEMV_IMPL=bdmma" "RELAX_Q4_GEMV_IMPL=mma"; do
  env $v timeout 100 python bench.py --no-cpu-baseline > gpurun_out/b.json 2>gpurun_out/b.err; a=$(val gpurun_out/b.json)
  env $v timeout 100 python bench.py --no-cpu-baseline --fused > gpurun_out/b.json 2>/dev/null; b=$(val gpurun_out/b.json)
  echo "$v: plain $a fused $b | l2 $(env $v python tools/l2_rate.py 4096 4096 | cut -d, -f1) $(env $v python tools/l2_rate.py 4096 11008 | cut -d, -f1)"
done
