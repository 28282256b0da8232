"""GPU parity of the measured-slower decode kernels kept for reference
(experiments build only: RELAX_Q4_GEMV_IMPL=mma|bdmma|row|v1, RELAX_Q4_GEMV_ZPF=0).

    python -m paper_2311_02103_b200.build --experiments
    python -m pytest experiments/tests -m gpu

The implementation switch is read once per process, so each one runs in a
subprocess against build_exp/librelax_q4_exp.so (RELAX_Q4_LIB):
experiments/tests/_gemv_impl_check.py compares it with the oracle on decode
shapes (n = 1, 2), including ragged K chunks and N smaller than one MMA row
block, plus the one-hot bitwise pin.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))


@pytest.mark.parametrize("impl,zpf", [("mma", "1"), ("bdmma", "1"), ("row", "1"), ("v1", "1"), ("stream", "0"), ("stream", "1")])
def test_gemv_impl_parity(impl, zpf):
    sys.path.insert(0, ROOT)
    from paper_2311_02103_b200 import build
    lib = build.build(experiments=True)
    env = dict(os.environ, RELAX_Q4_GEMV_IMPL=impl, RELAX_Q4_GEMV_ZPF=zpf, RELAX_Q4_LIB=lib)
    r = subprocess.run([sys.executable, os.path.join(HERE, "_gemv_impl_check.py")],
                       env=env, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "ALL OK" in r.stdout
