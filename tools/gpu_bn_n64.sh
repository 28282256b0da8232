#!/bin/bash
# Dispatch at 33 <= n <= 64: BN = 64 (the current choice) vs BN = 128 (half the tile idle), each with its automatic split
set -u
O=gpurun_out/bn64; mkdir -p $O; rm -f $O/s.jsonl
python -m paper_2311_02103_b200.build > $O/build.log 2>&1 || { echo BUILD_FAIL; exit 1; }
timeout 1500 python tools/sweep.py --shapes ${SHAPES:-4096x4096,11008x4096,4096x11008,4096x12288,4096x22016,4096x32000,5120x5120,13824x5120,5120x13824,8192x8192,28672x8192,8192x28672,8192x10240} \
   --ns ${NS:-24,33,40,48,56,64} --variants ${VARIANTS:-auto,tc::128,tc::64,tc::32} --out $O/s.jsonl > /dev/null 2>&1; echo "sweep rc=$?"
python - <<'PY'
import json
from collections import defaultdict
d=defaultdict(dict)
for l in open("gpurun_out/bn64/s.jsonl"):
    x=json.loads(l)
    if 'us' in x: d[(x['K'],x['N'],x['n'])][x['variant']]=x['us']
for k,v in sorted(d.items()):
    best=min(v,key=v.get)
    print(k, ' '.join(f"{a}={b:.2f}" for a,b in sorted(v.items())), "best", best, "x%.3f" % (v['auto']/v[best]))
PY
if [ "${TESTS:-0}" = "1" ]; then
  timeout 1500 python -m pytest tests/test_gpu_schedules.py tests/test_gpu_parity.py tests/test_gpu_fused.py -q --timeout 600 > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
fi
