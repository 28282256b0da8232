#!/usr/bin/env python3
"""Per-matrix kernel sweep: time each (K, N, n,
variant) as back-to-back calls in a CUDA graph that rotates over R distinct
weight copies totalling >= 4x the L2 (so weights stream from HBM), report
GB/s of algorithmic bytes and TFLOPS.  One JSON object per line.

    python tools/sweep.py [--shapes 4096x4096,...] [--ns 1,2,4,...] [--variants auto,gemv,tc,tc:4]
                          [--reps 20] [--out gpurun_out/sweep.jsonl] [--no-pdl]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2311_02103_b200 import inputs, ops  # noqa: E402

L2 = 126 * 2**20


def time_calls(fn_list, reps, stream):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for f in fn_list:
            f()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(reps):
            g.replay()
        e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (reps * len(fn_list))   # ms per call


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="4096x4096,4096x11008,11008x4096,4096x32000")
    ap.add_argument("--ns", default="1,2,3,4,6,8,12,16,24,32,48,64,96,128,256,512,1024,2048,4096")
    ap.add_argument("--variants", default="auto")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--min-bytes", type=float, default=4 * L2)
    ap.add_argument("--no-pdl", action="store_true")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "sweep.jsonl"))
    a = ap.parse_args()
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream()
    flags = ops.FLAG_NO_PDL if a.no_pdl else 0
    out = open(a.out, "a")
    for shp in a.shapes.split(","):
        K, N = map(int, shp.split("x"))
        wb = inputs.q4_bytes(K, N)
        R = int(min(256, max(1, np.ceil(a.min_bytes / wb))))
        pk, sc = inputs.realistic_weights(77 + K + N, K, N)
        pk_d = torch.from_numpy(pk.view(np.int32)).to(dev)
        sc_d = torch.from_numpy(sc.view(np.float16)).to(dev)
        copies = [(pk_d.clone(), sc_d.clone()) for _ in range(R)]
        del pk_d, sc_d
        for n in map(int, a.ns.split(",")):
            x = torch.from_numpy(inputs.activations(7 + n, n, K).view(np.float16)).to(dev)
            y = torch.empty((n, N), dtype=torch.float16, device=dev)
            ws = ops.workspace(n, K, N)
            for var in a.variants.split(","):
                if var == "gemv" and n > 8:
                    continue
                if var == "smalln" and n > 32:
                    continue
                base, _, sp = var.partition(":")        # "tc:S" forces split-K S (cluster reduction), "tc:S:BN" the tile
                sp, _, bnv = sp.partition(":")
                bn = int(bnv) if bnv else 0
                vflags = flags
                if base.endswith("-np"):                # one tile per CTA (no persistent kernel)
                    base = base[:-3]
                    vflags |= ops.FLAG_TILE_PER_CTA
                split = int(sp) if sp else 0
                v = {"auto": ops.VARIANT_AUTO, "gemv": ops.VARIANT_GEMV, "tc": ops.VARIANT_TC,
                     "smalln": ops.VARIANT_SMALLN}[base]
                # a rotation long enough to stream >= 4 L2 of weights per replay
                fns = [lambda p=p, s=s: ops.q4_matmul_ex(x, p, s, y=y, ws=ws, variant=v, flags=vflags,
                                                         split_k=split, bn=bn, stream=stream) for p, s in copies]
                try:
                    ms = time_calls(fns, a.reps, stream)
                except Exception as e:  # noqa: BLE001
                    print(json.dumps({"K": K, "N": N, "n": n, "variant": var, "error": str(e)}), flush=True)
                    continue
                by = wb + 2 * n * K + 2 * n * N
                rec = {"K": K, "N": N, "n": n, "variant": var, "split": split, "bn": bn,
                       "sched": ops.query_schedule(n, K, N),
                       "us": round(ms * 1e3, 3), "GBps": round(by / (ms * 1e-3) / 1e9, 1),
                       "TFLOPS": round(2 * n * K * N / (ms * 1e-3) / 1e12, 2), "R": R, "pdl": not a.no_pdl}
                print(json.dumps(rec), flush=True)
                out.write(json.dumps(rec) + "\n")
        del copies
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
