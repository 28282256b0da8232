#!/bin/bash
# A/B of the decode-chain timeline (tools/trace_step.py) against old_build/ (see tools/ab_tc.sh).
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
(cd old_build && python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1)
echo NEW; RELAX_Q4_TRACE=1 timeout 100 python tools/trace_step.py --layers 32 2>&1 | tail -1
echo OLD; (cd old_build && RELAX_Q4_TRACE=1 timeout 100 python ../tools/trace_step.py --layers 32 2>&1 | tail -1)
