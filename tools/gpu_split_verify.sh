set -u
O=gpurun_out/splv; mkdir -p $O
python -m paper_2311_02103_b200.build > $O/build.log 2>&1 || { echo BUILD_FAIL; exit 1; }
timeout 900 python -m pytest tests/test_gpu_schedules.py tests/test_gpu_parity.py -q --timeout 600 > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
for spec in "1024x8192 65,128" "1024x4096 256" "1024x1024 1024" "1024x2048 512"; do set -- $spec; timeout 300 python tools/sweep.py --shapes $1 --ns $2 --variants auto --out $O/s.jsonl > /dev/null 2>&1; done
python -c "
import json
for l in open('$O/s.jsonl'):
    d=json.loads(l); print(d['K'],d['N'],d['n'],d['sched'],d['us'])"
