#!/bin/bash
# A/B of the decode bench: this tree vs old_build/ (a snapshot of the previous commit)
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
(cd old_build && python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1)
val() { python -c "import json;d=json.load(open('$1'));print(d['value'])"; }
for i in 1 2; do
  for f in "" "--fused" "--n 2"; do
    timeout 100 python bench.py --no-cpu-baseline $f > gpurun_out/b_new.json 2>/dev/null
    (cd old_build && timeout 100 python bench.py --no-cpu-baseline $f > ../gpurun_out/b_old.json 2>/dev/null)
    echo "[$f] new: $(val gpurun_out/b_new.json)  old: $(val gpurun_out/b_old.json)"
  done
done
timeout 200 python bench.py --no-cpu-baseline --workload llama2-70b-decode > gpurun_out/b_new.json 2>/dev/null
(cd old_build && timeout 200 python bench.py --no-cpu-baseline --workload llama2-70b-decode > ../gpurun_out/b_old.json 2>/dev/null)
echo "[70b] new: $(val gpurun_out/b_new.json)  old: $(val gpurun_out/b_old.json)"
for sh in "4096 1024" "4096 4096" "4096 11008" "11008 4096"; do echo "new $(python tools/l2_rate.py $sh)"; (cd old_build && echo "old $(python tools/l2_rate.py $sh)"); done
