"""paper_2311_02103_b200 -- a B200-native fused q4f16 dequantize+matmul.

The hot path of Relax's LLM evaluation (arXiv 2311.02103): int4
weights, fp16 activations, y[n,N] = x[n,K] . dequant(Wq[K,N]) over a symbolic
token count n.  The compute runs in hand-written sm_100a CUDA behind a C-ABI
(include/relax_q4.h, built into paper_2311_02103_b200/librelax_q4.so); the
Python names here are argument marshalling only.

Submodules:
    ops      -- ctypes binding of the C-ABI (relax_q4_matmul, ...)
    inputs   -- seeded synthetic inputs (shared with the tests)
    tp       -- tensor-parallel sharding over torch.distributed
    build    -- nvcc build of the shared library
"""
__all__ = ["ops", "inputs", "tp", "build"]
