#!/usr/bin/env python3
"""Resident-cluster capacity of the tensor-core kernel per (BN, cluster size):
cudaOccupancyMaxActiveClusters through relax_debug_tc_max_clusters.

    python tools/tc_clusters.py
"""
import os
os.environ.setdefault("RELAX_Q4_LIB", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "build_exp", "librelax_q4_exp.so"))  # traces: experiments build
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402,F401
from paper_2311_02103_b200 import ops  # noqa: E402

L = ops.lib()
torch.cuda.init()
print("BN   " + " ".join(f"s={s:<5d}" for s in range(1, 9)) + "   (max resident clusters; CTAs = clusters * s)")
for bn in (16, 32, 64, 128, 256):
    print(f"{bn:<4d} " + " ".join(f"{L.relax_debug_tc_max_clusters(bn, s):<7d}" for s in range(1, 9)))
