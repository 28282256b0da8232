#!/usr/bin/env python3
"""Role wait-time breakdown of the tensor-core kernel (RELAX_Q4_TRACE=1).

    RELAX_Q4_TRACE=1 python tools/tc_trace.py K N n [variant_split] [bn]
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

REC = np.dtype([("cta", "<u4"), ("smid", "<u4"), ("nsub", "<u4"), ("pad", "<u4"), ("t0", "<u8"), ("te", "<u8"),
                ("w_prod", "<u8"), ("x_prod", "<u8"), ("perm", "<u8"), ("tr_w", "<u8"), ("tr_a", "<u8"),
                ("mma_a", "<u8"), ("mma_x", "<u8"), ("wst", "<u8"),
                ("t_mma0", "<u8"), ("t_acc", "<u8"), ("t_epi", "<u8"),
                ("t_cb1", "<u8"), ("t_cred", "<u8"), ("t_cb2", "<u8")])
K, N, n = map(int, sys.argv[1:4])
split = int(sys.argv[4]) if len(sys.argv) > 4 else 0
bn = int(sys.argv[5]) if len(sys.argv) > 5 else 0
L = ops.lib()
L.relax_debug_tctrace_read.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t), ctypes.c_int]
pk, sc = inputs.stress_weights(K + N, K, N)
pw = torch.from_numpy(pk.view(np.int32)).cuda()
s = torch.from_numpy(sc.view(np.float16)).cuda()
x = torch.from_numpy(inputs.activations(1, n, K).view(np.float16)).cuda()
y = torch.empty((n, N), dtype=torch.float16, device="cuda")
for _ in range(3):
    ops.q4_matmul_ex(x, pw, s, y=y, variant=ops.VARIANT_TC, split_k=split, bn=bn)
torch.cuda.synchronize()
buf = np.zeros(1 << 14, dtype=REC)
cnt = ctypes.c_size_t(0)
L.relax_debug_tctrace_read(buf.ctypes.data, buf.size, ctypes.byref(cnt), 1)
ops.q4_matmul_ex(x, pw, s, y=y, variant=ops.VARIANT_TC, split_k=split, bn=bn)
torch.cuda.synchronize()
L.relax_debug_tctrace_read(buf.ctypes.data, buf.size, ctypes.byref(cnt), 1)
r = buf[:cnt.value]
dur = (r["te"] - r["t0"]) / 1e3
print(f"K={K} N={N} n={n} sched={ops.query_schedule(n, K, N)} ctas={len(r)} nsub={r['nsub'][0]}")
print(f"CTA duration us: min {dur.min():.2f} med {np.median(dur):.2f} max {dur.max():.2f}; "
      f"kernel span {(r['te'].max() - r['t0'].min()) / 1e3:.2f} us")
st = (r["t0"] - r["t0"].min()) / 1e3
print(f"CTA start offset us: p10 {np.percentile(st, 10):.2f} p50 {np.median(st):.2f} p90 {np.percentile(st, 90):.2f} "
      f"max {st.max():.2f}; CTAs per SM histogram {np.bincount(np.bincount(r['smid'].astype(np.int64)))}")
ph = lambda a_, b_: np.median((r[b_].astype(np.int64) - r[a_].astype(np.int64)) / 1e3)  # noqa: E731
print(f"phases (median us): start->first MMA {ph('t0', 't_mma0'):.2f}  first MMA->acc ready {ph('t_mma0', 't_acc'):.2f}  "
      f"acc ready->stores done {ph('t_acc', 't_epi'):.2f}  stores done->exit {ph('t_epi', 'te'):.2f}")
if r["t_cb1"].max() > 0:
    print(f"cluster split (median us): acc ready->after barrier 1 {ph('t_acc', 't_cb1'):.2f}  reduce+store {ph('t_cb1', 't_cred'):.2f}  "
          f"barrier 2 {ph('t_cred', 't_cb2'):.2f}")
for f in ["w_prod", "x_prod", "perm", "tr_w", "tr_a", "mma_a", "mma_x", "wst"]:
    us = r[f] / 1.9e3
    print(f"  wait {f:7s}: median {np.median(us):7.2f} us  max {us.max():7.2f} us   (cycles/1.9GHz)")
