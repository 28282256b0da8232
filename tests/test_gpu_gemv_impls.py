"""GPU parity of the non-default decode kernels (RELAX_Q4_GEMV_IMPL=mma|row|v1).

The implementation switch is read once per process, so each one runs in a
subprocess: tests/_gemv_impl_check.py compares it with the oracle on decode
shapes (n = 1, 2), including ragged K chunks and N smaller than one MMA row
block, plus the one-hot bitwise pin.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("impl", ["mma", "bdmma", "row", "v1"])
def test_gemv_impl_parity(impl):
    env = dict(os.environ, RELAX_Q4_GEMV_IMPL=impl)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "_gemv_impl_check.py")],
                       env=env, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "ALL OK" in r.stdout
