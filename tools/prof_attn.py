#!/usr/bin/env python3
"""One decode-attention configuration, a few calls -- the target of ncu.
    python tools/prof_attn.py batch Hq Hkv L [reps]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2311_02103_b200 import ops  # noqa: E402

b, hq, hkv, L = (int(v) for v in sys.argv[1:5])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 5
q = torch.randn((b, hq, 128), device="cuda").half()
k = torch.randn((b, hkv, L, 128), device="cuda").half()
v = torch.randn((b, hkv, L, 128), device="cuda").half()
lens = torch.full((b,), L, dtype=torch.int32, device="cuda")
out = torch.empty_like(q)
ws = torch.empty(ops.attn_decode_workspace(b, hq, L), dtype=torch.uint8, device="cuda")
for _ in range(reps):
    ops.attn_decode(q, k, v, lens, out=out, ws=ws)
torch.cuda.synchronize()
# 20 calls captured in a CUDA graph (device time, no host dispatch in it)
st = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=st):
    for _ in range(20):
        ops.attn_decode(q, k, v, lens, out=out, ws=ws, stream=st)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(st):
    g.replay()
    e0.record(st)
    g.replay()
    e1.record(st)
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / 20
byts = 2 * b * hkv * L * 128 * 2
print(f"attention b={b} Hq={hq} Hkv={hkv} L={L}: {us:.1f} us/call, {byts / us / 1e3:.0f} GB/s (KV bytes)")
