#!/bin/bash
# Fixed-latency breakdown of the decode GEMV (profiles/gemv_latency_r01.txt): needs exp_build/, a copy of
# the package whose gemv_stream.cu honours -DEXP_NO_X / -DEXP_NO_WAIT and whose build.py passes $EXP_DEFS.
cd exp_build
for v in "" "-DEXP_NO_X" "-DEXP_NO_WAIT" "-DEXP_NO_X -DEXP_NO_WAIT"; do
  rm -rf build paper_2311_02103_b200/librelax_q4.so
  EXP_DEFS="$v" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
  echo "== variant [$v]"
  for sh in "4096 1024" "4096 4096" "4096 11008"; do python tools/l2_rate.py $sh; done
done
