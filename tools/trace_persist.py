#!/usr/bin/env python3
"""Per-CTA segment timeline of the persistent tensor-core kernel (experiments
build, RELAX_Q4_TRACE=1): for each CTA its start, and per segment (pair tile p,
stages [kb0, kb1)) the time the accumulator was ready, the partial written,
all partials of the tile in, and the segment done; then the CTA end.  Times in
us from the earliest CTA start.

    RELAX_Q4_LIB=build_exp/librelax_q4_exp.so RELAX_Q4_TRACE=1 \\
        python tools/trace_persist.py K N n [--all]
"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2311_02103_b200 import inputs, ops  # noqa: E402

SEGS = 8
WORDS = 3 + SEGS * 5 + 1


def main():
    K, N, n = map(int, sys.argv[1:4])
    show_all = "--all" in sys.argv
    pk, sc = inputs.realistic_weights(5 + K + N, K, N)
    pw = torch.from_numpy(pk.view(np.int32)).cuda()
    s = torch.from_numpy(sc.view(np.float16)).cuda()
    x = torch.from_numpy(inputs.activations(7 + n, n, K).view(np.float16)).cuda()
    ws = ops.workspace(n, K, N)
    y = torch.empty((n, N), dtype=torch.float16, device="cuda")
    for _ in range(4):
        ops.q4_matmul_ex(x, pw, s, y=y, ws=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ops.q4_matmul_ex(x, pw, s, y=y, ws=ws)
    e1.record()
    torch.cuda.synchronize()
    buf = np.zeros(512 * WORDS, dtype=np.uint64)
    L = ops.lib()
    L.relax_debug_ptrace_read.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
    assert L.relax_debug_ptrace_read(buf.ctypes.data, buf.nbytes) == 0
    q = ops.query_schedule(n, K, N)
    print(f"K={K} N={N} n={n} sched={q} event time {e0.elapsed_time(e1) * 1e3:.1f} us")
    t = buf.reshape(512, WORDS)
    ctas = [i for i in range(512) if t[i, 2] != 0]
    t0 = min(int(t[i, 2]) for i in ctas)
    us = lambda v: (int(v) - t0) / 1e3 if v else float("nan")  # noqa: E731
    ends = []
    for i in ctas:
        nseg = int(t[i, 0]) >> 32
        sm = int(t[i, 0]) & 0xFFFFFFFF
        row = f"cta {i:3d} cl {int(t[i, 1]):3d} sm {sm:3d} start {us(t[i, 2]):7.2f} |"
        for g in range(min(nseg, SEGS)):
            w = int(t[i, 3 + g * 5])
            p, kb0, kb1 = w & 0xFFFFFFFF, (w >> 32) & 0xFFFF, (w >> 48) & 0xFFFF
            st = [us(t[i, 4 + g * 5 + k]) for k in range(4)]
            row += f" p{p}[{kb0},{kb1}) acc {st[0]:.1f} part {st[1]:.1f} all {st[2]:.1f} done {st[3]:.1f} |"
        row += f" end {us(t[i, WORDS - 1]):.2f}"
        ends.append(us(t[i, WORDS - 1]))
        if show_all or i % 8 == 0:
            print(row)
    ends = np.array(ends)
    print(f"CTA end us: min {ends.min():.1f} median {np.median(ends):.1f} max {ends.max():.1f}; "
          f"first start to last end {ends.max():.1f} us over {len(ctas)} CTAs")


if __name__ == "__main__":
    main()
