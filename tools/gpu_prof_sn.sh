#!/bin/bash
O=gpurun_out/prof_sn; mkdir -p $O
for spec in "4096 32000 8" "11008 4096 8"; do
  set -- $spec
  tag=${1}x${2}_n$3
  timeout 120 python tools/prof_one.py $1 $2 $3 smalln 5 > /dev/null 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:smalln -s 2 -c 1 -o $O/sn_$tag python tools/prof_one.py $1 $2 $3 smalln 5 > $O/ncu_$tag.log 2>&1
  echo "ncu $tag rc=$?"
  bash tools/ncu_summary.sh $O/sn_$tag.ncu-rep > $O/sum_$tag.txt 2>&1; cat $O/sum_$tag.txt
done
