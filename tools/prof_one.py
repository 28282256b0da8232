#!/usr/bin/env python3
"""Run one (K, N, n, variant) configuration a few times -- the target for
`ncu --set full` (one GPU, short).  python tools/prof_one.py K N n [variant] [reps]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2311_02103_b200 import inputs, ops  # noqa: E402

K, N, n = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
var = {"auto": 0, "gemv": 1, "tc": 2, "smalln": 3}[sys.argv[4] if len(sys.argv) > 4 else "auto"]
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 5
pk, sc = inputs.realistic_weights(5 + K + N, K, N)
pw = torch.from_numpy(pk.view(np.int32)).cuda()
s = torch.from_numpy(sc.view(np.float16)).cuda()
x = torch.from_numpy(inputs.activations(7 + n, n, K).view(np.float16)).cuda()
ws = ops.workspace(n, K, N)
y = torch.empty((n, N), dtype=torch.float16, device="cuda")
for _ in range(reps):
    ops.q4_matmul_ex(x, pw, s, y=y, ws=ws, variant=var)
torch.cuda.synchronize()
print("ok", K, N, n, ops.query_schedule(n, K, N))
