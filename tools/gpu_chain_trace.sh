python -m paper_2311_02103_b200.build --experiments > /dev/null 2>&1 || echo BUILDFAIL
RELAX_Q4_LIB=build_exp/librelax_q4_exp.so timeout 300 python tools/chain_trace.py 2>&1 | tail -45 | head -12
