#!/bin/bash
# A/B of where the decode GEMV signals griddepcontrol.launch_dependents (RELAX_Q4_GS_TRIGGER).
set -u
O=gpurun_out/trig; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "zero_invariants or one_hot or config1" > $O/pytest_zero.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_zero.log
for rep in 1 2; do
for t in 0 1 2; do
  for spec in "7b:" "7bfused:--fused" "70b:--workload llama2-70b-decode"; do
    tag=${spec%%:*}; fl=${spec#*:}
    RELAX_Q4_GS_TRIGGER=$t timeout 600 python bench.py $fl --no-cpu-baseline > $O/b_${tag}_t${t}_r$rep.json 2> $O/b_${tag}_t${t}_r$rep.err
    echo "trig=$t $tag rep=$rep: $(python -c "import json,sys; d=json.load(open('$O/b_${tag}_t${t}_r$rep.json')); print(d['value'], d['roofline']['frac'], d['clocks'])" 2>&1 | tail -1)"
  done
done
done
