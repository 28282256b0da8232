#!/bin/bash
# Decoder-block benches (bench.py --block fused|unfused) for 7B and 13B.
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
val() { python -c "import json;d=json.load(open('$1'));print(d['value'], d['ms_per_step'], d['e2e']['value'], d['gpu_launches'], d['config']['workload'])"; }
for b in "--fused" "--block fused" "--block unfused"; do
  timeout 200 python bench.py --no-cpu-baseline $b > gpurun_out/blk.json 2> gpurun_out/blk.err; echo "$b rc=$?: $(val gpurun_out/blk.json 2>&1 | tail -1)"; tail -2 gpurun_out/blk.err
done
timeout 200 python bench.py --no-cpu-baseline --block fused --workload llama2-13b-decode > gpurun_out/blk.json 2>/dev/null; echo "13b fused: $(val gpurun_out/blk.json)"
timeout 200 python bench.py --no-cpu-baseline --block unfused --workload llama2-13b-decode > gpurun_out/blk.json 2>/dev/null; echo "13b unfused: $(val gpurun_out/blk.json)"
