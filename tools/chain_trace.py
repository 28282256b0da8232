"""Per-op timeline of the persistent decode chain (experiments build, RQ4_TRACE):
    RELAX_Q4_LIB=build_exp/librelax_q4_exp.so python tools/chain_trace.py [workload]
Prints, for the first ops of the 7B layer set, the median / max over CTAs of
each phase and the spread of completion times."""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2311_02103_b200 import inputs, ops  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "llama2-7b-decode"
model, mats = bench.layer_set(wl)
dev = torch.device("cuda", 0)
proto = {}
for i, (K, N) in enumerate(sorted({(K, N) for _, K, N in mats})):
    pk, sc = inputs.realistic_weights(2000 + i, K, N)
    proto[(K, N)] = (torch.from_numpy(pk.view(np.int32)).to(dev), torch.from_numpy(sc.view(np.float16)).to(dev))
W = [(proto[(K, N)][0].clone(), proto[(K, N)][1].clone()) for _, K, N in mats]
xs = {K: torch.from_numpy(inputs.activations(7 + K, 1, K).view(np.float16)).to(dev) for K in {K for _, K, _ in mats}}
ys = [torch.empty((1, N), dtype=torch.float16, device=dev) for _, _, N in mats]
heads = ("q", "o", "gate", "down", "lm_head")
ch = ops.DecodeChain([(xs[K], *W[j], ys[j], nm.split(".")[-1] in heads) for j, (nm, K, N) in enumerate(mats)])
for _ in range(3):
    ch.run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
ch.run()
e1.record()
torch.cuda.synchronize()
print(f"{wl}: {len(mats)} ops, one launch {e0.elapsed_time(e1) * 1e3:.1f} us")
L = ops.lib()
buf = np.zeros(160 * 256 * 7, dtype=np.uint64)
L.relax_debug_chain_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
assert L.relax_debug_chain_trace_read(buf.ctypes.data, buf.nbytes) == 0
sms = torch.cuda.get_device_properties(0).multi_processor_count
tr = buf.reshape(160, 256, 7)[:sms].astype(np.int64)
t0 = tr[:, 0, 0].min()
print("op  name              start(us)  wait  xload (ld)  stages  epi+sig  done_spread  prod_first(us)")
for m in range(min(len(mats), 40)):
    r = tr[:, m, :] - t0
    st = np.median(r[:, 0]) / 1e3
    wait = np.median(r[:, 1] - r[:, 0]) / 1e3
    xl = np.median(r[:, 2] - r[:, 1]) / 1e3
    xld = np.median(r[:, 6] - r[:, 1]) / 1e3
    sg = np.median(r[:, 3] - r[:, 2]) / 1e3
    ep = np.median(r[:, 4] - r[:, 3]) / 1e3
    spread = (r[:, 4].max() - r[:, 4].min()) / 1e3
    pf = np.median(r[:, 5]) / 1e3
    print(f"{m:3d} {mats[m][0]:16s} {st:9.2f} {wait:6.2f} {xl:6.2f} ({xld:5.2f}) {sg:7.2f} {ep:8.2f} {spread:11.2f} {pf:10.2f}")
