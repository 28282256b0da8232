#!/usr/bin/env python3
"""Per-CTA timeline of the small-batch decode chain (n = 3..8; experiments
build, RELAX_Q4_TRACE=1): the first L layers of the Llama-2-7B set with
q/k/v and gate/up as grouped launches, replayed from a CUDA graph.

    RELAX_Q4_LIB=build_exp/librelax_q4_exp.so RELAX_Q4_TRACE=1 python tools/trace_smalln.py [--layers 3] [--n 8]
"""
import argparse
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("RELAX_Q4_TRACE", "1")
os.environ.setdefault("RELAX_Q4_LIB", os.path.join(ROOT, "build_exp", "librelax_q4_exp.so"))
from paper_2311_02103_b200 import inputs, ops  # noqa: E402

REC = np.dtype([("seq", "<u4"), ("cta", "<u4"), ("p0", "<u4"), ("p1", "<u4"),
                ("t0", "<u8"), ("tw", "<u8"), ("tf", "<u8"), ("te0", "<u8"), ("te", "<u8")])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=3)
    ap.add_argument("--n", type=int, default=8)
    a = ap.parse_args()
    L = ops.lib()
    L.relax_debug_sntrace_read.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t), ctypes.c_int]
    spec = inputs.LLAMA_SETS["llama2-7b"]
    mats = [(nm, K, N) for _ in range(a.layers) for nm, K, N in spec["mats"]]
    dev = torch.device("cuda", 0)
    ws = []
    for nm, K, N in mats:
        pk, sc = inputs.stress_weights(K + N, K, N)
        ws.append((torch.from_numpy(pk.view(np.int32)).to(dev), torch.from_numpy(sc.view(np.float16)).to(dev)))
    xs = {K: torch.from_numpy(inputs.activations(K, a.n, K).view(np.float16)).to(dev) for _, K, _ in mats}
    ys = [torch.empty((a.n, N), dtype=torch.float16, device=dev) for _, _, N in mats]
    groups, i = [], 0
    while i < len(mats):
        kind = mats[i][0].split(".")[-1]
        span = 3 if kind == "q" else 2 if kind == "gate" else 1
        groups.append(list(range(i, i + span)))
        i += span
    st = torch.cuda.Stream()

    def step():
        for g in groups:
            if len(g) == 1:
                j = g[0]
                ops.q4_matmul(xs[mats[j][1]], *ws[j], y=ys[j], stream=st)
            else:
                ops.q4_matmul_grouped(xs[mats[g[0]][1]], [ws[j] for j in g], ys=[ys[j] for j in g], stream=st)
    with torch.cuda.stream(st):
        step()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=st):
        step()
    with torch.cuda.stream(st):
        for _ in range(3):
            gr.replay()
    torch.cuda.synchronize()
    buf = np.zeros(1 << 16, dtype=REC)
    n = ctypes.c_size_t(0)
    L.relax_debug_sntrace_read(buf.ctypes.data, buf.size, ctypes.byref(n), 1)
    with torch.cuda.stream(st):
        gr.replay()
    torch.cuda.synchronize()
    L.relax_debug_sntrace_read(buf.ctypes.data, buf.size, ctypes.byref(n), 1)
    r = buf[:n.value]
    seqs = sorted(set(r["seq"].tolist()))
    T0 = r["t0"].min()
    print(f"{'launch':>6} {'shape':>12} {'ctas':>4} | {'start min/max':>15} | {'wait':>6} {'first':>6} {'epi':>6} | "
          f"{'end min/max':>15} | {'stages':>6} {'epi':>5}  (us)")
    for k, sq in enumerate(seqs):
        q = r[r["seq"] == sq]
        g = groups[k % len(groups)]
        K, N = mats[g[0]][1], sum(mats[j][2] for j in g)
        us = lambda v: (v - T0) / 1e3  # noqa: E731
        print(f"{sq:>6} {K:>5}x{N:<6} {len(q):>4} | {us(q['t0'].min()):7.2f} {us(q['t0'].max()):7.2f} | "
              f"{np.median(q['tw'] - q['t0']) / 1e3:6.2f} {np.median(q['tf'] - q['t0']) / 1e3:6.2f} "
              f"{np.median(q['te0'] - q['t0']) / 1e3:6.2f} | {us(q['te'].min()):7.2f} {us(q['te'].max()):7.2f} | "
              f"{np.median(q['te0'] - q['tf']) / 1e3:6.2f} {np.median(q['te'] - q['te0']) / 1e3:5.2f}")
    tot = (r["te"].max() - T0) / 1e3
    print(f"total {tot:.2f} us for {len(groups)} launches")


if __name__ == "__main__":
    main()
