#!/bin/bash
# A/B of tensor-core sweeps: this tree vs old_build/ (a snapshot of an earlier commit: copy the
# package, include/, oracle/, bench.py and tools/sweep.py, summarize_sweep.py into old_build/ first).
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
(cd old_build && python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1)
A="--shapes 4096x4096,11008x4096 --ns 128,512,2048 --variants auto --reps 10"
timeout 300 python tools/sweep.py $A --out gpurun_out/tc_new.jsonl > /dev/null 2>&1
(cd old_build && timeout 300 python tools/sweep.py $A --out ../gpurun_out/tc_old.jsonl > /dev/null 2>&1)
echo NEW; python tools/summarize_sweep.py gpurun_out/tc_new.jsonl | grep "^| [0-9]"
echo OLD; python tools/summarize_sweep.py gpurun_out/tc_old.jsonl | grep "^| [0-9]"
for w in "--workload llama2-70b-decode"; do
  timeout 200 python bench.py --no-cpu-baseline $w > gpurun_out/b.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/b.json'));print('new', '$w', d['value'])"
done
