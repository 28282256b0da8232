#!/usr/bin/env python3
"""Per-CTA timeline of one decode step (RELAX_Q4_TRACE=1 builds the trace).

    RELAX_Q4_TRACE=1 python tools/trace_step.py [--layers 2] [--out gpurun_out/trace.txt]

Runs the first L layers of the Llama-2-7B decode set (7 GEMVs per layer) as a
CUDA graph, replays it, reads the per-CTA records (globaltimer ns) and prints,
per launch: CTA start spread, time waiting for the previous kernel
(griddepcontrol.wait), first-stage arrival, end spread.
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
from paper_2311_02103_b200 import inputs, ops  # noqa: E402

REC = np.dtype([("seq", "<u4"), ("cta", "<u4"), ("smid", "<u4"), ("pad", "<u4"),
                ("t0", "<u8"), ("tw", "<u8"), ("tf", "<u8"), ("te", "<u8")])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=2)
    ap.add_argument("--no-pdl", action="store_true")
    ap.add_argument("--grouped", action="store_true", help="q/k/v and gate/up as grouped launches (the bench default)")
    a = ap.parse_args()
    L = ops.lib()
    L.relax_debug_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_size_t,
                                         ctypes.POINTER(ctypes.c_size_t), ctypes.c_int]
    spec = inputs.LLAMA_SETS["llama2-7b"]
    mats = [(nm, K, N) for _ in range(a.layers) for nm, K, N in spec["mats"]]
    dev = torch.device("cuda", 0)
    ws = []
    for nm, K, N in mats:
        pk, sc = inputs.stress_weights(K + N, K, N)
        ws.append((torch.from_numpy(pk.view(np.int32)).to(dev), torch.from_numpy(sc.view(np.float16)).to(dev)))
    xs = {K: torch.from_numpy(inputs.activations(K, 1, K).view(np.float16)).to(dev) for _, K, _ in mats}
    ys = [torch.empty((1, N), dtype=torch.float16, device=dev) for _, _, N in mats]
    st = torch.cuda.Stream()
    flags = ops.FLAG_NO_PDL if a.no_pdl else 0

    groups, i = [], 0
    while i < len(mats):
        kind = mats[i][0].split(".")[-1]
        span = (3 if kind == "q" else 2 if kind == "gate" else 1) if a.grouped else 1
        groups.append(list(range(i, i + span)))
        i += span

    def step():
        for g in groups:
            if len(g) == 1:
                j = g[0]
                ops.q4_matmul_ex(xs[mats[j][1]], *ws[j], y=ys[j], flags=flags, stream=st)
            else:
                ops.q4_matmul_grouped(xs[mats[g[0]][1]], [ws[j] for j in g], ys=[ys[j] for j in g], stream=st)
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
    L.relax_debug_trace_read(buf.ctypes.data, buf.size, ctypes.byref(n), 1)   # reset
    g.replay()
    torch.cuda.synchronize()
    L.relax_debug_trace_read(buf.ctypes.data, buf.size, ctypes.byref(n), 1)
    r = buf[:n.value]
    seqs = sorted(set(r["seq"].tolist()))
    T0 = r["t0"].min()
    print(f"{'seq':>4} {'shape':>12} {'ctas':>4} | {'start min/max':>15} | {'wait_rel':>9} {'first_rel':>9} | "
          f"{'end min/max':>15} | {'x->end':>7} {'first->epi':>10} {'epi':>6}  (us, rel. to step start)")
    prev_end = None
    for i, s in enumerate(seqs):
        q = r[r["seq"] == s]
        g = groups[i % len(groups)]
        K = mats[g[0]][1]
        N = sum(mats[j][2] for j in g)
        us = lambda v: (v - T0) / 1e3  # noqa: E731
        line = (f"{s:>4} {K:>5}x{N:<6} {len(q):>4} | {us(q['t0'].min()):7.2f} {us(q['t0'].max()):7.2f} | "
                f"{np.median(q['tw'] - q['t0']) / 1e3:9.2f} {np.median(q['tf'] - q['t0']) / 1e3:9.2f} | "
                f"{us(q['te'].min()):7.2f} {us(q['te'].max()):7.2f} | {np.median(q['te'] - q['tw']) / 1e3:7.2f}"
                f" {np.median(q['t0'] + q['pad'] - q['tf']) / 1e3:10.2f} {np.median(q['te'] - q['t0'] - q['pad']) / 1e3:6.2f}"
                f"  sm/cta {len(set(q['smid'].tolist()))}/{np.bincount(q['smid']).max()}")
        print(line)
        prev_end = q["te"].max()
    tot = (r["te"].max() - T0) / 1e3
    byts = sum(inputs.q4_bytes(K, N) for _, K, N in mats)
    print(f"total {tot:.2f} us for {len(mats)} GEMVs, {byts / 1e6:.1f} MB -> {byts / (tot * 1e-6) / 1e9:.0f} GB/s")


if __name__ == "__main__":
    main()
