#!/bin/bash
# Decode bench under GEMV knob settings (used for the prefetch-depth experiment).
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
val() { python -c "import json;d=json.load(open('$1'));print(d['value'])"; }
for v in "X=1" "RELAX_Q4_GS_L2PF=0" "X=1" "RELAX_Q4_GS_L2PF=0"; do
  env $v timeout 100 python bench.py --no-cpu-baseline > gpurun_out/b.json 2>/dev/null; a=$(val gpurun_out/b.json)
  env $v timeout 100 python bench.py --no-cpu-baseline --fused > gpurun_out/b.json 2>/dev/null; b=$(val gpurun_out/b.json)
  env $v timeout 200 python bench.py --no-cpu-baseline --workload llama2-70b-decode > gpurun_out/b.json 2>/dev/null; c=$(val gpurun_out/b.json)
  echo "$v: plain $a fused $b 70b $c"
done
