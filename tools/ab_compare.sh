#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
(cd old_build && python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1)
val() { python -c "import json;d=json.load(open('$1'));print(d['value'])"; }
for i in 1 2; do
  timeout 100 python bench.py --no-cpu-baseline $BENCH_ARGS > gpurun_out/b_new.json 2>/dev/null; echo "new: $(val gpurun_out/b_new.json)"
  (cd old_build && timeout 100 python bench.py --no-cpu-baseline $BENCH_ARGS > ../gpurun_out/b_old.json 2>/dev/null); echo "old: $(val gpurun_out/b_old.json)"
done
for sh in "4096 4096" "4096 11008" "11008 4096" "4096 32000"; do python tools/l2_rate.py $sh; done
(cd old_build && for sh in "4096 4096" "4096 11008" "11008 4096" "4096 32000"; do python tools/l2_rate.py $sh; done)
