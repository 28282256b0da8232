#!/usr/bin/env python3
"""Measured one-wave capacity of split-K clusters: for each cluster size s,
the largest tile count whose tiles * s CTAs all start in the first wave
(no SM runs more than its resident CTAs, no late starters), from the
per-CTA trace (RELAX_Q4_TRACE=1).  cudaOccupancyMaxActiveClusters
under-reports this at two CTAs per SM (tools/tc_clusters.py).

    RELAX_Q4_TRACE=1 python tools/tc_waves.py [bn]
"""
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

REC = np.dtype([("cta", "<u4"), ("smid", "<u4"), ("nsub", "<u4"), ("pad", "<u4"), ("t0", "<u8"), ("te", "<u8")]
               + [(f"f{i}", "<u8") for i in range(14)])
L = ops.lib()
L.relax_debug_tctrace_read.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t), ctypes.c_int]
bn = int(sys.argv[1]) if len(sys.argv) > 1 else 16
per_sm = 2 if bn <= 64 else 1
n = min(bn, 8) if bn <= 64 else bn
K = 256 * 16
buf = np.zeros(1 << 14, dtype=REC)
cnt = ctypes.c_size_t(0)


def one_wave(tiles, s):
    N = 128 * tiles
    pk, sc = inputs.stress_weights(7, K, N)
    pw = torch.from_numpy(pk.view(np.int32)).cuda()
    sv = torch.from_numpy(sc.view(np.float16)).cuda()
    x = torch.from_numpy(inputs.activations(1, n, K).view(np.float16)).cuda()
    y = torch.empty((n, N), dtype=torch.float16, device="cuda")
    ok = True
    for _ in range(3):
        L.relax_debug_tctrace_read(buf.ctypes.data, buf.size, ctypes.byref(cnt), 1)
        ops.q4_matmul_ex(x, pw, sv, y=y, variant=ops.VARIANT_TC, split_k=s, bn=bn)
        torch.cuda.synchronize()
        L.relax_debug_tctrace_read(buf.ctypes.data, buf.size, ctypes.byref(cnt), 1)
        r = buf[:cnt.value]
        assert len(r) == tiles * s, (len(r), tiles, s)
        dur = (r["te"] - r["t0"]).min()
        late = (r["t0"] - r["t0"].min()).max()
        ok = ok and np.bincount(r["smid"].astype(np.int64)).max() <= per_sm and late < 0.5 * dur
    return ok


print(f"BN={bn} ({per_sm} CTA/SM), K={K}: largest one-wave tile count per cluster size s")
for s in range(2, 9):
    hi = (per_sm * 148) // s
    t = hi
    while t > 1 and not one_wave(t, s):
        t -= 1
    print(f"s={s}: {t} clusters ({t * s} CTAs; slot bound {hi})", flush=True)
