#!/usr/bin/env python3
"""Per-CTA timeline of the decoder-block chain (bench.py --block fused|unfused)
for the first L layers, from the GEMV trace (RELAX_Q4_TRACE=1).

    RELAX_Q4_TRACE=1 python tools/trace_block.py [--layers 2] [--block fused]
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
os.environ.setdefault("RELAX_Q4_LIB", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "build_exp", "librelax_q4_exp.so"))  # traces: experiments build
import bench  # noqa: E402
from paper_2311_02103_b200 import inputs, ops  # noqa: E402

REC = np.dtype([("seq", "<u4"), ("cta", "<u4"), ("smid", "<u4"), ("pad", "<u4"),
                ("t0", "<u8"), ("tw", "<u8"), ("tf", "<u8"), ("te", "<u8")])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=2)
    ap.add_argument("--block", default="fused")
    a = ap.parse_args()
    L = ops.lib()
    L.relax_debug_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t), ctypes.c_int]
    _, mats = bench.layer_set("llama2-7b-decode", fused=True)
    mats = mats[:4 * a.layers] + mats[-1:]
    dev = torch.device("cuda", 0)
    weights = []
    for nm, K, N in mats:
        pk, sc = inputs.stress_weights(K + N, K, N)
        weights.append((torch.from_numpy(pk.view(np.int32)).to(dev), torch.from_numpy(sc.view(np.float16)).to(dev)))
    st = torch.cuda.Stream()
    args = argparse.Namespace(block=a.block, workload="llama2-7b-decode")
    step, _ = bench.block_step(args, mats, weights, 1, dev, st)
    with torch.cuda.stream(st):
        step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        step()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    buf = np.zeros(1 << 16, dtype=REC)
    n = ctypes.c_size_t(0)
    L.relax_debug_trace_read(buf.ctypes.data, buf.size, ctypes.byref(n), 1)
    g.replay()
    torch.cuda.synchronize()
    L.relax_debug_trace_read(buf.ctypes.data, buf.size, ctypes.byref(n), 1)
    r = buf[:n.value]
    seqs = sorted(set(r["seq"].tolist()))
    T0 = r["t0"].min()
    print(f"{'seq':>4} {'name':>10} {'shape':>12} | {'start min/max':>15} | {'wait_rel':>9} {'x_rel':>9} | "
          f"{'end min/max':>15} | {'wait->end':>9}")
    for i, s in enumerate(seqs):
        q = r[r["seq"] == s]
        nm, K, N = mats[i % len(mats)]
        us = lambda v: (v - T0) / 1e3  # noqa: E731
        print(f"{s:>4} {nm:>10} {K:>5}x{N:<6} | {us(q['t0'].min()):7.2f} {us(q['t0'].max()):7.2f} | "
              f"{np.median(q['tw'] - q['t0']) / 1e3:9.2f} {np.median(q['tf'] - q['t0']) / 1e3:9.2f} | "
              f"{us(q['te'].min()):7.2f} {us(q['te'].max()):7.2f} | {np.median(q['te'] - q['tw']) / 1e3:9.2f}")
    print(f"total {(r['te'].max() - T0) / 1e3:.2f} us for {len(seqs)} GEMV launches")


if __name__ == "__main__":
    main()
