#!/bin/bash
# Stream-K of the persistent kernel (experiments build: RELAX_Q4_STREAMK=1, full waves whole + the rest
# cut into k units, deferred fixups) vs the product's schedules (=0); product parity of the persistent
# path; a product sweep of the persistent shapes.
set -u
O=gpurun_out/sk; mkdir -p $O
python -m paper_2311_02103_b200.build > $O/build.log 2>&1 || { echo BUILD_FAIL; exit 1; }
python -m paper_2311_02103_b200.build --experiments > $O/build_exp.log 2>&1 || { echo BUILD_EXP_FAIL; exit 1; }
RELAX_Q4_LIB=build_exp/librelax_q4_exp.so RELAX_Q4_STREAMK=1 timeout 600 python -m pytest tests/test_gpu_streamk.py -q -x --timeout 300 > $O/pytest_sk.log 2>&1; echo "pytest streamk (exp) rc=$?"; tail -2 $O/pytest_sk.log
timeout 1500 python -m pytest tests/test_gpu_schedules.py tests/test_gpu_threads.py tests/test_gpu_parity.py tests/test_gpu_large.py tests/test_gpu_streamk.py -q --timeout 900 > $O/pytest_product.log 2>&1; echo "pytest product rc=$?"; tail -2 $O/pytest_product.log
timeout 900 python tools/sweep.py --shapes 4096x11008,4096x32000,11008x4096,4096x22016 --ns 1024,2048,4096 --variants auto --out $O/sweep_product.jsonl > /dev/null 2>&1; echo "sweep product rc=$?"
python -c "
import json
for l in open('$O/sweep_product.jsonl'):
    d=json.loads(l); print(d['K'],d['N'],d['n'],d['sched'],d['us'],d['TFLOPS'])"
