"""Subprocess body for experiments/tests/test_gpu_gemv_impls.py (needs a GPU).

Runs the decode path (n = 1, 2, forced GEMV variant) under whatever
RELAX_Q4_GEMV_IMPL the parent set and checks it against the oracle.
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_2311_02103_b200 import inputs, ops  # noqa: E402
from tests._util import assert_within_tol, dev_weights, dev_x, host_bits  # noqa: E402

SHAPES = [(256, 256), (256, 5), (512, 17), (2048, 300), (2304, 160), (4096, 1000), (11008, 700), (4352, 40)]


def main():
    for i, (K, N) in enumerate(SHAPES):
        for kind in ("realistic", "stress"):
            packed, scales = inputs.weights(kind, 3000 + i, K, N)
            pw, sc = dev_weights(packed, scales)
            for n in (1, 2):
                xb = inputs.activations(11 + n + i, n, K, "normal" if kind == "realistic" else "uniform")
                r = oracle.matmul_f64(xb, packed, scales, K, N)
                y = torch.full((n, N), float("nan"), dtype=torch.float16, device="cuda")
                ops.q4_matmul_ex(dev_x(xb), pw, sc, y=y, variant=ops.VARIANT_GEMV)
                torch.cuda.synchronize()
                assert_within_tol(host_bits(y), r, f"{os.environ.get('RELAX_Q4_GEMV_IMPL')} {kind} K={K} N={N} n={n}")
        # one-hot rows extract W bitwise (pins the in-kernel dequant)
        packed, scales = inputs.weights("stress", 3100 + i, K, N)
        pw, sc = dev_weights(packed, scales)
        w = oracle.dequant(packed, scales, K, N)           # fp16 bits [N][K]
        for k in (0, K // 3, K - 1):
            xb = np.zeros((1, K), dtype=np.uint16)
            xb[0, k] = 0x3C00
            y = torch.empty((1, N), dtype=torch.float16, device="cuda")
            ops.q4_matmul_ex(dev_x(xb), pw, sc, y=y, variant=ops.VARIANT_GEMV)
            torch.cuda.synchronize()
            got = host_bits(y)[0]
            want = w[:, k]
            assert np.array_equal(got, want), \
                f"one-hot K={K} N={N} k={k}"
    print("ALL OK")


if __name__ == "__main__":
    main()
