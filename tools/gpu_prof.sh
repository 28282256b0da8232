#!/bin/bash
# Sweep + ncu captures (each profiled command first runs plain and must exit 0).
set -u
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD_FAIL; exit 1; }
if [ -n "${SWEEP_ARGS:-}" ]; then
  rm -f gpurun_out/sweep.jsonl
  timeout 900 python tools/sweep.py $SWEEP_ARGS > gpurun_out/sweep.log 2>&1; echo "sweep rc=$?"; tail -3 gpurun_out/sweep.log
fi
i=0
for spec in ${PROF_SPECS:-}; do   # spec = K:N:n:variant:kregex
  IFS=: read K N n v kr <<< "$spec"
  i=$((i+1))
  timeout 120 python tools/prof_one.py $K $N $n $v 5 > gpurun_out/prof_plain_$i.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$kr -s 2 -c 1 \
      -o gpurun_out/prof_${K}x${N}_n${n}_${v} python tools/prof_one.py $K $N $n $v 5 > gpurun_out/ncu_$i.log 2>&1
  echo "prof $spec rc=$?"; tail -2 gpurun_out/ncu_$i.log
done
if [ -n "${LAUNCH_LIST:-}" ]; then
  timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ll_plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv \
      --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_ll.log 2>&1
  echo "launch list rc=$?"; tail -2 gpurun_out/ncu_ll.log
fi
