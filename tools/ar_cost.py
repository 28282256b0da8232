"""Per-call cost of the fused row-split all-reduce epilogue (relax_q4_matmul_allreduce)
at NCCL world 1 vs the plain decode kernel, in a PDL chain captured in a CUDA graph."""
import os
import socket
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_02103_b200 import inputs, ops, tp  # noqa: E402

s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
torch.cuda.set_device(0)
dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                        device_id=torch.device("cuda", 0))
ex = tp.TpExchange(8192)
st = torch.cuda.Stream()
for K, N in [(4096, 4096), (11008, 4096), (1024, 8192), (3584, 8192), (512, 4096)]:
    R = 40
    ws = []
    for i in range(R):
        pk, sc = inputs.realistic_weights(50 + (i % 3), K, N)
        ws.append((torch.from_numpy(pk.view(np.int32)).cuda(), torch.from_numpy(sc.view(np.float16)).cuda()))
    x = torch.from_numpy(inputs.activations(1, 1, K).view(np.float16)).cuda()
    y = torch.empty((1, N), dtype=torch.float16, device="cuda")
    res = {}
    for mode in ("plain", "allreduce", "plain+nccl"):
        def chain():
            for w in ws:
                if mode == "allreduce":
                    ops.q4_matmul_allreduce(x, *w, ex.comm, y=y, stream=st)
                elif mode == "plain":
                    ops.q4_matmul(x, *w, y=y, stream=st)
                else:
                    ops.q4_matmul(x, *w, y=y, stream=st)
                    y32 = y.float()
                    dist.all_reduce(y32)
                    y.copy_(y32)
        with torch.cuda.stream(st):
            chain()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            chain()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            for _ in range(3):
                g.replay()
            torch.cuda.synchronize()
            e0.record(st)
            for _ in range(20):
                g.replay()
            e1.record(st)
        torch.cuda.synchronize()
        res[mode] = e0.elapsed_time(e1) * 1e3 / (20 * R)
    print(f"K={K} N={N}: " + "  ".join(f"{m} {v:.2f} us" for m, v in res.items()), flush=True)
dist.destroy_process_group()
