#!/usr/bin/env python3
"""Math-rate probe of the decode GEMV: one L2-resident weight matrix called
back to back (CUDA graph, PDL) so the stream never waits on HBM and the time
per call is the kernel's compute + latency floor.

    python tools/l2_rate.py [K N [calls]]
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2311_02103_b200 import inputs, ops  # noqa: E402


def main():
    K = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    N = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
    calls = int(sys.argv[3]) if len(sys.argv) > 3 else 200
    pk, sc = inputs.realistic_weights(77, K, N)
    pw = torch.from_numpy(pk.view(np.int32)).cuda()
    s = torch.from_numpy(sc.view(np.float16)).cuda()
    x = torch.from_numpy(inputs.activations(5, 1, K).view(np.float16)).cuda()
    y = torch.empty((1, N), dtype=torch.float16, device="cuda")
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        ops.q4_matmul_ex(x, pw, s, y=y, stream=st)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for _ in range(calls):
            ops.q4_matmul_ex(x, pw, s, y=y, stream=st)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        e0.record(st)
        for _ in range(5):
            g.replay()
        e1.record(st)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / (5 * calls)
    byts = inputs.q4_bytes(K, N)
    print(f"K={K} N={N}: {us:.2f} us/call, {byts / us / 1e3:.0f} GB/s (L2-resident), "
          f"{K * N / (us * 1e-6) / 148 / 1.9e9:.1f} weights/clk/SM at 1.9 GHz")


if __name__ == "__main__":
    main()
