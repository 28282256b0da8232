"""Streaming rate of the decode chain with no dependencies: `count` ops of one
shape, all reading the same x (no waits, x kept in registers) -- the
consumer compute rate vs HBM.  python tools/chain_rate.py K N count [after_every]"""
import os
import sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_02103_b200 import inputs, ops  # noqa: E402

K, N, cnt = (int(v) for v in sys.argv[1:4])
every = int(sys.argv[4]) if len(sys.argv) > 4 else 0
pk, sc = inputs.realistic_weights(3, K, N)
pw = torch.from_numpy(pk.view(np.int32)).cuda()
sw = torch.from_numpy(sc.view(np.float16)).cuda()
W = [(pw.clone(), sw.clone()) for _ in range(cnt)]
x = torch.from_numpy(inputs.activations(4, 1, K).view(np.float16)).cuda()
ys = [torch.empty((1, N), dtype=torch.float16, device="cuda") for _ in range(cnt)]
ch = ops.DecodeChain([(x, *W[i], ys[i], bool(every) and i % every == 0 and i > 0) for i in range(cnt)])
for _ in range(3):
    ch.run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    ch.run()
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / 5
byt = cnt * (N * K // 2 + N * K // 16)
print(f"chain {cnt} x {K}x{N} after_every={every}: {us:.1f} us, {byt / us / 1e3:.0f} GB/s, {us / cnt:.2f} us/op")
